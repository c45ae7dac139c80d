/*
 * dtq_capi.h -- C ABI of the B200 (sm_100a) quantized-linear path.
 *
 * This is the drop-in boundary for the reference's L1 numerics core
 * (/root/reference/proj/core/include/dtq/{quant,balance,qgemm,plan}.hpp).
 * Plain pointers, sizes and status codes only: no C++ or torch types.
 * Every device-side entry point is stream-ordered on the given CUDA stream
 * (`stream` is a cudaStream_t passed as void*; NULL = legacy default) and
 * never synchronises unless documented.  Device pointers are marked [dev],
 * host pointers [host].
 *
 * Status codes mirror the reference's exception types:
 *   DTQ_OK                    success
 *   DTQ_ERR_INVALID_ARGUMENT  std::invalid_argument (shape/bits/non-finite)
 *   DTQ_ERR_OVERFLOW          std::overflow_error (accumulator bound)
 *   DTQ_ERR_CUDA              CUDA runtime/driver failure
 *   DTQ_ERR_UNSUPPORTED       std::logic_error (not available on this build)
 * dtq_last_error() returns the calling thread's last message.
 *
 * There is no CPU fallback: without a sm_100 device every compute entry
 * point fails with DTQ_ERR_CUDA.
 */
#ifndef DTQ_CAPI_H
#define DTQ_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DTQ_CAPI_VERSION 1

typedef enum dtq_status {
  DTQ_OK = 0,
  DTQ_ERR_INVALID_ARGUMENT = 1,
  DTQ_ERR_OVERFLOW = 2,
  DTQ_ERR_CUDA = 3,
  DTQ_ERR_UNSUPPORTED = 4
} dtq_status;

/* element types of activations / outputs */
typedef enum dtq_dtype {
  DTQ_F16 = 0,
  DTQ_BF16 = 1,
  DTQ_F32 = 2,
  DTQ_F64 = 3,
  DTQ_S32 = 4 /* output only: zero-point-corrected integer accumulator */
} dtq_dtype;

/* arithmetic of the activation quantizer */
typedef enum dtq_mode {
  /* fp32 transforms; codes/s/z bit-identical to the reference when no
   * prologue, smoothing or rotation is applied (tie-guarded fp64 divide) */
  DTQ_MODE_FAST = 0,
  /* fp64 transforms in the reference's operation order: bit-identical to
   * the reference with smoothing and rotation as well */
  DTQ_MODE_EXACT = 1
} dtq_mode;

/* prologue fused in front of the quantizer (one HBM pass) */
typedef enum dtq_prologue_kind {
  DTQ_PROLOGUE_NONE = 0,
  DTQ_PROLOGUE_MODULATE = 1,    /* x*(1+scale[c])+shift[c]   toydit.cpp:339-369 */
  DTQ_PROLOGUE_GELU = 2,        /* 0.5x(1+erf(x/sqrt2))      toydit.cpp:83      */
  DTQ_PROLOGUE_LN_MODULATE = 3  /* LayerNorm (no affine, eps) then modulate;
                                   no reference oracle: parity unpinned      */
} dtq_prologue_kind;

typedef struct dtq_prologue {
  int32_t kind;        /* dtq_prologue_kind */
  const float* scale;  /* [dev] [K] (MODULATE / LN_MODULATE) */
  const float* shift;  /* [dev] [K] */
  float eps;           /* LN_MODULATE */
} dtq_prologue;

/* BalanceTransform (balance.hpp:31-34): mask then rotation, both optional.
 * The rotation is blockwise: I_{K/hblock} (x) (D * H_hblock / sqrt(hblock)),
 * which is the reference rotate_channels when hblock == K. */
typedef struct dtq_balance {
  const double* smooth; /* [dev] [K] ScalingMask.s (X / s, W * s) or NULL     */
  const int8_t* signs;  /* [dev] [K] RotationMatrix.sign_diag (+-1) or NULL   */
  int32_t hblock;       /* rotation block, power of two in [8, 16384]; blocks
                           wider than 256 take an fp64 pre-pass (exact)      */
} dtq_balance;

/* opaque quantized-linear handle (QuantLinear, qgemm.hpp:17-24) */
typedef struct dtq_qlinear_s* dtq_qlinear_t;

/* ---------------------------------------------------------------- misc */
const char* dtq_last_error(void);
int dtq_capi_version(void);
/* 0 if a usable sm_100 device is current, else DTQ_ERR_CUDA */
int dtq_device_check(void);

/* ---------------------------------------------------------------- quantizer
 * quantize(x, per_token | per_output_channel, bits, Dynamic, nullptr,
 * symmetric)  -- replaces quant.hpp:94-97 / quant.cpp:140-177 for the row
 * groupings (one (s, z) per row), with an optional fused prologue and
 * channel balance in front.
 *   x       [dev] rows x cols of x_dtype, row pitch ldx elements
 *   codes   [dev] rows x cols u8, row pitch ldc bytes
 *   scale   [dev] rows f64 (QuantParams.scale)
 *   zero    [dev] rows i32 (QuantParams.zero_point)
 *   status  [dev] optional i32; |= 1 if any input is non-finite (the
 *           reference throws std::invalid_argument; the stream-ordered API
 *           reports it here instead of synchronising)
 * bits in {2,4,6,8}.  Tie rounding is half-to-even (quant.cpp:9-16). */
int dtq_quantize_rows(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                      int bits, int symmetric, int mode, const dtq_balance* balance,
                      const dtq_prologue* prologue, uint8_t* codes, int64_t ldc,
                      double* scale, int32_t* zero, int32_t* status, void* stream);

/* ---------------------------------------------------------------- weights
 * make_quant_linear (qgemm.cpp:9-21) on the device, with the weight side of
 * apply_balance (W * diag(s), then the same rotation; balance.cpp:126-140,
 * dtq_main.cpp:276-290) fused in front, all in fp64 as the reference.
 *   w        [dev] N x K of w_dtype (F16/BF16/F32/F64), pitch ldw elements
 *   bias     [dev] N f64 or NULL
 *   balance  NULL or the layer's transform (copied into the handle; the
 *            forward applies the activation side automatically)
 * weight_bits and act_bits in {2,4,6,8}.  W4 weights are stored packed (two
 * codes per byte, trace_io.cpp:79-91 nibble order) and unpacked in shared
 * memory by the GEMM; 2-, 6- and 8-bit weights are stored as s8 w_sym. */
int dtq_qlinear_create(const void* w, int w_dtype, int64_t N, int64_t K, int64_t ldw,
                       int weight_bits, int act_bits, const double* bias,
                       const dtq_balance* balance, void* stream, dtq_qlinear_t* out);

/* Build from already-quantized weights (checkpoint loader path,
 * trace_io.cpp:263-316): reference codes in [0, 2^b-1] with z = 2^(b-1).
 *   codes   [dev] packed==0: N x K u8, pitch ld bytes
 *                 packed==1: trace_io LSB-first bit stream of N*K codes
 *   scale   [dev] N f64 */
int dtq_qlinear_create_from_codes(const uint8_t* codes, int packed, int64_t ld,
                                  int weight_bits, const double* scale, int64_t N, int64_t K,
                                  int act_bits, const double* bias, const dtq_balance* balance,
                                  void* stream, dtq_qlinear_t* out);

int dtq_qlinear_destroy(dtq_qlinear_t h);

int dtq_qlinear_info(dtq_qlinear_t h, int64_t* N, int64_t* K, int* weight_bits,
                     int* act_bits);

/* Copy the prepared weights back for inspection:
 *   codes [host] N x K u8 reference codes (w_sym + z_w), scale [host] N f64,
 *   wsum [host] N i32 (sum_c w_sym, qgemm.cpp:44-48).  Any may be NULL.
 * Synchronises `stream`. */
int dtq_qlinear_export(dtq_qlinear_t h, uint8_t* codes, double* scale, int32_t* wsum,
                       void* stream);

/* ---------------------------------------------------------------- GEMM
 * qlinear_forward core (qgemm.cpp:52-63) on quantized activations:
 *   codes [dev] M x K u8 with row pitch ldc (a multiple of 16 bytes)
 *   s_x, z_x [dev] per-token params from dtq_quantize_rows
 *   y [dev] M x N of y_dtype, pitch ldy elements:
 *     F16 / BF16 / F32 : s_x*s_w*acc + bias, fp32 epilogue
 *     S32              : acc - z_x*wsum (exact integer, for parity)
 *     F64              : the reference's fp64 epilogue, bit-identical
 *                        (uses an internal M x N s32 scratch)
 * Fails with DTQ_ERR_OVERFLOW when (2^act_bits-1) * 2^(wbits-1) * K does
 * not fit int32 (K > 65793 at W8A8), mirroring qgemm.cpp:29-34. */
int dtq_qgemm(const uint8_t* codes, int64_t ldc, const double* s_x, const int32_t* z_x,
              int64_t M, dtq_qlinear_t h, void* y, int y_dtype, int64_t ldy, void* stream);

/* ---------------------------------------------------------------- fused layer
 * Whole Matrix qlinear_forward(x, layer) (qgemm.cpp:23-67) on the device:
 * fused quantizer (prologue + the handle's balance) then the GEMM.
 * `workspace` [dev] of dtq_qlinear_workspace_bytes(h, M) bytes (row-flag
 * counters, codes and per-token params; for a W4A8 handle also its weights
 * expanded to s8, N x round_up(K, 16) bytes, which the quantizer writes and
 * the W8A8 GEMM reads; 16-byte aligned), or NULL to use a handle-owned
 * buffer.  A caller workspace must be zero-filled before its first use (its
 * first 33 KB are the counters through which the GEMM consumes row blocks as
 * the concurrently running quantizer publishes them); every forward leaves
 * them zero again.  Calls that use
 * handle-owned scratch (workspace NULL, or y_dtype DTQ_F64, whose s32
 * accumulator is handle-owned) must be ordered on one stream or serialised
 * by the caller; with a caller workspace and a non-F64 output, calls on one
 * handle may run concurrently on different streams. */
size_t dtq_qlinear_workspace_bytes(dtq_qlinear_t h, int64_t M);
int dtq_qlinear_forward(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                        int mode, const dtq_prologue* prologue, void* y, int y_dtype,
                        int64_t ldy, void* workspace, size_t workspace_bytes,
                        int32_t* status, void* stream);

/* dtq_qlinear_forward with an activation applied to y in the GEMM's epilogue,
 * on the fp32 value before the cast: DTQ_ACT_GELU gives
 * gelu(qlinear_forward(x)) (toydit.cpp:83) in the same pass -- the fc1 ->
 * gelu step of toydit.cpp:215-216, so the next layer's quantizer runs with no
 * prologue.  F16 / BF16 outputs (else DTQ_ERR_UNSUPPORTED). */
typedef enum dtq_activation { DTQ_ACT_NONE = 0, DTQ_ACT_GELU = 1 } dtq_activation;
int dtq_qlinear_forward_act(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                            int mode, const dtq_prologue* prologue, int activation, void* y,
                            int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes,
                            int32_t* status, void* stream);

/* The quantizer stage of dtq_qlinear_forward alone: the activation side of
 * the handle's balance (X / s with the handle's fp32 reciprocals in FAST
 * mode, fp64 divide in EXACT mode, then the rotation) + optional prologue +
 * per-token quantization at the handle's act_bits.  codes [dev] M x K u8
 * with pitch ldc (multiple of 16 for the GEMM), scale/zero [dev] M. */
int dtq_qlinear_quantize(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                         int mode, const dtq_prologue* prologue, uint8_t* codes, int64_t ldc,
                         double* scale, int32_t* zero, int32_t* status, void* stream);

/* Same with HOST buffers (x [host] M x K dense, y [host] M x N dense):
 * H2D copy, fused forward, D2H copy, stream synchronised before returning.
 * From 1024 rows (non-F64 outputs) the rows run as a pipeline of chunks of
 * 128, 256, 512, ... rows on three internal streams (H2D / forward / D2H), so
 * the D2H of early chunks overlaps the rest.  Pinned host memory gives full
 * PCIe/C2C bandwidth.  Non-finite input is
 * reported as DTQ_ERR_INVALID_ARGUMENT (the reference's exception).
 * Thread-safe: concurrent calls on one handle are serialised (the handle
 * owns the staging buffers and streams). */
int dtq_qlinear_forward_host(const void* x, int x_dtype, int64_t M, dtq_qlinear_t h, int mode,
                             void* y, int y_dtype, void* stream);

/* ---------------------------------------------------------------- fp64 parity kernels
 * Device implementations of the remaining reference operations, in fp64 and
 * in the reference's operation order (bit-identical results).  Used by the
 * C++ drop-in (the include/dtq/ headers); not on the timed path.
 *
 * grouping: 0 PerTensor, 1 PerToken, 2 PerChannel, 3 PerOutputChannel,
 *           4 PerGroup(group_size)   (quant.hpp:26-48 GroupingScheme::kind)
 * scale/zero: one entry per group, [dev]. */
int dtq_quantize_static(const double* x, int64_t rows, int64_t cols, int64_t ldx, int bits,
                        int grouping, int64_t group_size, const double* scale,
                        const int32_t* zero, uint8_t* codes, int64_t ldc, void* stream);

/* out = s * (code - z)   (quant.cpp:179-188) */
int dtq_dequantize(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ldc, int grouping,
                   int64_t group_size, const double* scale, const int32_t* zero, double* out,
                   int64_t ldo, void* stream);

/* apply_scaling / rotate_channels (balance.cpp:57-67, 94-107) on rows:
 * out = [x * s | x / s] then, per hblock columns, signs, FWHT, 1/sqrt(hb).
 * smooth and signs may each be NULL; hblock a power of two <= 16384. */
int dtq_balance_apply(const double* x, int64_t rows, int64_t cols, int64_t ldx,
                      const double* smooth, int smooth_mul, const int8_t* signs, int64_t hblock,
                      double* out, int64_t ldo, void* stream);

/* y = x * w^T (+ bias) in fp64 with the reference's sequential summation
 * (matrix.hpp:62-76): the qlinear_forward_float oracle path. */
int dtq_matmul_nt_f64(const double* x, int64_t M, int64_t K, const double* w, int64_t N,
                      const double* bias, double* y, void* stream);

/* Calibration statistics (matrix.hpp:95-109): out[c] = max_r |x[r,c]|
 * (col, out [dev] cols) / out[r] = max_c |x[r,c]| (row, out [dev] rows). */
int dtq_col_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                       void* stream);
int dtq_row_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                       void* stream);

/* fwht (balance.cpp:22-33) in place on each of `rows` rows of n values
 * (n a power of two <= 16384): the unnormalised radix-2 butterflies in the
 * reference's order, no signs, no 1/sqrt(n). */
int dtq_fwht_f64(double* x, int64_t rows, int64_t n, int64_t ldx, void* stream);

/* ---------------------------------------------------------------- checkpoints
 * read_checkpoint (trace_io.cpp:263-316) straight onto the device.  The
 * file is the reference's little-endian format: "DTQCKPT\0", u16 version 1,
 * u32 layer count, then per layer the name, shape, bits, grouping, symmetric
 * flag, f32 scales (+ i32 zero points when asymmetric), the codes packed
 * LSB-first (trace_io.cpp:79-91), the f32 scaling mask and the rotation
 * signs as bits.  Bad magic / version / truncation / trailing bytes fail
 * with DTQ_ERR_INVALID_ARGUMENT (the reference's FormatError). */
typedef struct dtq_checkpoint_s* dtq_checkpoint_t;

int dtq_checkpoint_open(const char* path, dtq_checkpoint_t* out);
int dtq_checkpoint_close(dtq_checkpoint_t ck);
int dtq_checkpoint_num_layers(dtq_checkpoint_t ck, int64_t* n);

/* Layer i: name (NUL-terminated, owned by ck), C_out, C_in, weight bits,
 * symmetric flag, mask length and rotation length (0 = none). */
int dtq_checkpoint_layer_info(dtq_checkpoint_t ck, int64_t i, const char** name, int64_t* N,
                              int64_t* K, int* bits, int* symmetric, int64_t* mask_len,
                              int64_t* rot_len);

/* Device-resident quantized linear of layer i.  The packed codes are
 * uploaded as stored and unpacked on the device (W4: straight into the
 * GEMM's nibble layout); the f32 scales become the fp64 s_w exactly as
 * read_checkpoint widens them; the mask becomes the smoothing vector and the
 * rotation signs the rotation over the stored rotation length (the weights
 * were rotated by that full rot_len-point Hadamard); `hblock` must be 0 or
 * equal to it (anything else is DTQ_ERR_INVALID_ARGUMENT).  Needs symmetric
 * per-output-channel weights (the GEMM's layout): anything else is
 * DTQ_ERR_UNSUPPORTED. */
int dtq_checkpoint_load_layer(dtq_checkpoint_t ck, int64_t i, int act_bits, int hblock,
                              void* stream, dtq_qlinear_t* out);

/* ---------------------------------------------------------------- mixed precision
 * One layer of a MixedPrecisionPlan (plan.hpp:30-40): the weight bits of each
 * of the kNumRanges = 4 timestep ranges.  The layer keeps one device-resident
 * QuantLinear per distinct bit width in its row (e.g. W8 for range 0, W4 for
 * ranges 1-3), all built from the same weights and balance by
 * dtq_qlinear_create.  The forward of denoising step t of `steps` dispatches
 * to bits_for(layer, t * 4 / steps), the range index of toydit.cpp:113-117.
 *   bits [host] 4 entries in {2,4,6,8} (the reference's 16 = floating-point
 *        passthrough is not a quantized layer: DTQ_ERR_INVALID_ARGUMENT) */
typedef struct dtq_planned_s* dtq_planned_t;

int dtq_planned_create(const void* w, int w_dtype, int64_t N, int64_t K, int64_t ldw,
                       const int32_t* bits, int act_bits, const double* bias,
                       const dtq_balance* balance, void* stream, dtq_planned_t* out);
int dtq_planned_destroy(dtq_planned_t p);
/* the handle serving denoising step t of `steps` (borrowed: owned by p);
 * steps >= 1, 0 <= t < steps, else DTQ_ERR_INVALID_ARGUMENT */
int dtq_planned_select(dtq_planned_t p, int64_t t, int64_t steps, dtq_qlinear_t* out);
/* weight bits of range r (0..3) */
int dtq_planned_bits(dtq_planned_t p, int r, int* bits);

#ifdef __cplusplus
}
#endif
#endif /* DTQ_CAPI_H */
