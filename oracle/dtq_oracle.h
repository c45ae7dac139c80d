/*
 * dtq_oracle.h -- CPU restatement of the reference quantized-linear path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product library
 * (paper_2406_02540_b200/libdtq_b200.so) never links or calls it.
 *
 * Every function restates the reference algorithm in plain C and cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * It is pinned against the real reference (oracle/_ref/libdtq_ref.so, built
 * from the reference sources by oracle/Makefile) and against the committed
 * golden vectors in tests/golden/ (see tests/test_oracle.py).
 *
 * Status codes: 0 ok, 1 invalid argument (std::invalid_argument in the
 * reference), 2 overflow (std::overflow_error).
 */
#ifndef DTQ_ORACLE_H
#define DTQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* core/src/quant.cpp:9-16 */
double dtq_oracle_round_even(double v);

/* core/src/quant.cpp:90-113 (asymmetric, zero-inclusive, degenerate s=1) */
int dtq_oracle_minmax_params(const double* g, int64_t n, int bits, double* s, int32_t* z);

/* core/src/quant.cpp:115-124 (z = 2^(b-1), s = max|x| / (2^(b-1)-1)) */
int dtq_oracle_symmetric_params(const double* g, int64_t n, int bits, double* s, int32_t* z);

/* quantize(x, per_token | per_output_channel, bits, Dynamic, nullptr, symmetric)
 * core/src/quant.cpp:140-177; one group per row. */
int dtq_oracle_quantize_rows(const double* x, int64_t rows, int64_t cols, int bits,
                             int symmetric, uint8_t* codes, double* s, int32_t* z);

/* Static quantize with one frozen (s, z) per row: quant.cpp:169-175. */
int dtq_oracle_quantize_rows_static(const double* x, int64_t rows, int64_t cols, int bits,
                                    const double* s, const int32_t* z, uint8_t* codes);

/* dequantize: quant.cpp:179-188  out = s * (code - z) */
void dtq_oracle_dequantize_rows(const uint8_t* codes, int64_t rows, int64_t cols,
                                const double* s, const int32_t* z, double* out);

/* balance.cpp:22-33 unnormalized radix-2 FWHT, h = 1, 2, 4, ... */
int dtq_oracle_fwht(double* d, int64_t n);

/* balance.cpp:69-80: sign_diag[c] = (mt19937_64(seed)() & 1) ? +1 : -1,
 * n draws in channel order (randomize=true), all +1 otherwise. */
void dtq_oracle_hadamard_signs(int64_t n, int randomize, uint64_t seed, int8_t* out);

/* Blockwise rotation: per hblock-wide column block j, the reference
 * rotate_channels (balance.cpp:94-107) with RotationMatrix{hblock,
 * signs[j*hblock:(j+1)*hblock]}.  hblock == cols reduces to the reference
 * exactly.  hblock must be a power of two >= 2 dividing cols. */
int dtq_oracle_rotate_blocks(double* x, int64_t rows, int64_t cols, int64_t hblock,
                             const int8_t* signs);

/* balance.cpp:35-55 */
int dtq_oracle_scaling_mask(const double* act_amax, const double* w_amax, int64_t n,
                            double alpha, double* s_out);

/* balance.cpp:57-67: X' = X / s (per column), W' = W * s */
void dtq_oracle_scale_x(double* x, int64_t rows, int64_t cols, const double* s);
void dtq_oracle_scale_w(double* w, int64_t rows, int64_t cols, const double* s);

/* toydit.cpp:366-368: out = x * (1 + scale[c]) + shift[c] */
void dtq_oracle_modulate(double* x, int64_t rows, int64_t cols, const double* scale,
                         const double* shift);

/* toydit.cpp:83: 0.5 x (1 + erf(x / sqrt 2)) */
void dtq_oracle_gelu(double* x, int64_t n);
/* LayerNorm over each row, no affine (the LN of the north_star's LN-modulate
 * prologue).  The reference has no LayerNorm: semantics of
 * torch.nn.functional.layer_norm (biased variance, eps inside the sqrt),
 * pinned against it in fp64 by tests/test_oracle.py. */
void dtq_oracle_layernorm(double* x, int64_t rows, int64_t cols, double eps);

/* qgemm.cpp:29-34 int64 overflow guard: returns 2 if it would throw. */
int dtq_oracle_overflow_guard(int act_bits, int weight_bits, int64_t c_in);

/* qgemm.cpp:40-60 corrected integer accumulator
 *   acc[t,o] = sum_c x[t,c] * (w[o,c] - z_w[o]) - z_x[t] * sum_c (w[o,c] - z_w[o])
 * computed in int64 exactly as the reference. `threads` <= 0 means all. */
int dtq_oracle_qlinear_acc(const uint8_t* xc, const int32_t* zx, int64_t M, int64_t K,
                           const uint8_t* wc, const int32_t* zw, int64_t N, int64_t* acc,
                           int threads);

/* host cores online (the CPU-baseline thread count) */
int dtq_oracle_num_cpus(void);

/* std::mt19937_64(seed), n-th output (1-based); pins the sign generator */
uint64_t dtq_oracle_mt19937_64_nth(uint64_t seed, int64_t n);

/* qgemm.cpp:61-63 epilogue y = s_x[t] * s_w[o] * (double)acc (+ bias[o]) */
void dtq_oracle_qlinear_epilogue(const int64_t* acc, const double* sx, int64_t M,
                                 const double* sw, const double* bias, int64_t N,
                                 double* y);

/* Whole qlinear_forward (qgemm.cpp:23-67) from float x and prepared weight
 * codes/params: quantize per token, int64 dot, correction, epilogue. */
int dtq_oracle_qlinear_forward(const double* x, int64_t M, int64_t K, int act_bits,
                               const uint8_t* wc, const double* sw, const int32_t* zw,
                               int weight_bits, int64_t N, const double* bias, double* y,
                               int threads);

/* trace_io.cpp:79-109 LSB-first code packing; returns packed byte count or -1 */
int64_t dtq_oracle_pack_codes(const uint8_t* codes, int64_t count, int bits, uint8_t* out);
int dtq_oracle_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count,
                            uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
