/*
 * dtq_oracle.c -- CPU restatement of the reference quantized-linear path.
 *
 * TEST INFRASTRUCTURE ONLY (see dtq_oracle.h).  Never linked into the
 * product library; used by tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs as the checker.
 *
 * Citations are to /root/reference/proj.  The arithmetic is kept in the
 * reference's order (fp64 everywhere, round-half-to-even, int64
 * accumulation) so the results are bit-identical to the reference; the
 * parity of this file with the reference itself is asserted by
 * tests/test_oracle.py against oracle/_ref/libdtq_ref.so and the golden
 * vectors in tests/golden/.
 */
#include "dtq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#include <pthread.h>
#include <unistd.h>

static int bits_supported(int bits) {
  /* quant.cpp:18-20 */
  return bits == 2 || bits == 4 || bits == 6 || bits == 8;
}

static double clampd(double v, double lo, double hi) {
  /* std::clamp(v, lo, hi): (v < lo) ? lo : (hi < v) ? hi : v */
  return (v < lo) ? lo : ((hi < v) ? hi : v);
}

double dtq_oracle_round_even(double v) {
  /* quant.cpp:9-16 */
  const double fl = floor(v);
  const double frac = v - fl;
  if (frac < 0.5) return fl;
  if (frac > 0.5) return fl + 1.0;
  return (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;
}

static int check_group(const double* g, int64_t n, int bits) {
  /* quant.cpp:50-58 */
  if (n <= 0) return 1;
  if (!bits_supported(bits)) return 1;
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(g[i])) return 1;
  return 0;
}

int dtq_oracle_minmax_params(const double* g, int64_t n, int bits, double* s, int32_t* z) {
  /* quant.cpp:90-113 */
  if (check_group(g, n, bits)) return 1;
  double mn = g[0], mx = g[0];
  for (int64_t i = 1; i < n; ++i) {
    if (g[i] < mn) mn = g[i];
    if (!(g[i] < mx)) mx = g[i];
  }
  const double qmax = (double)((1 << bits) - 1);
  if (mx == mn) {
    /* degenerate constant group: quant.cpp:97-104 */
    *s = 1.0;
    *z = (int32_t)clampd(dtq_oracle_round_even(-mn), 0.0, qmax);
    return 0;
  }
  /* widen to include zero: quant.cpp:107-108 (std::min / std::max) */
  const double lo = (0.0 < mn) ? 0.0 : mn;
  const double hi = (mx < 0.0) ? 0.0 : mx;
  *s = (hi - lo) / qmax;
  *z = (int32_t)clampd(dtq_oracle_round_even(-lo / *s), 0.0, qmax);
  return 0;
}

int dtq_oracle_symmetric_params(const double* g, int64_t n, int bits, double* s, int32_t* z) {
  /* quant.cpp:115-124 */
  if (check_group(g, n, bits)) return 1;
  double amax = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double a = fabs(g[i]);
    if (amax < a) amax = a;
  }
  *z = 1 << (bits - 1);
  *s = amax > 0.0 ? amax / (double)((1 << (bits - 1)) - 1) : 1.0;
  return 0;
}

static void quantize_row(const double* x, int64_t cols, double s, int32_t z, double qmax,
                         uint8_t* out) {
  /* quant.cpp:169-175 */
  for (int64_t c = 0; c < cols; ++c) {
    const double k = dtq_oracle_round_even(x[c] / s) + z;
    out[c] = (uint8_t)clampd(k, 0.0, qmax);
  }
}

int dtq_oracle_quantize_rows(const double* x, int64_t rows, int64_t cols, int bits,
                             int symmetric, uint8_t* codes, double* s, int32_t* z) {
  /* quant.cpp:140-177, Dynamic mode, PerToken / PerOutputChannel grouping */
  if (!bits_supported(bits)) return 1;
  if (rows <= 0 || cols <= 0) return 1;
  for (int64_t i = 0; i < rows * cols; ++i)
    if (!isfinite(x[i])) return 1;
  const double qmax = (double)((1 << bits) - 1);
  for (int64_t r = 0; r < rows; ++r) {
    const double* row = x + r * cols;
    const int st = symmetric ? dtq_oracle_symmetric_params(row, cols, bits, &s[r], &z[r])
                             : dtq_oracle_minmax_params(row, cols, bits, &s[r], &z[r]);
    if (st) return st;
    quantize_row(row, cols, s[r], z[r], qmax, codes + r * cols);
  }
  return 0;
}

int dtq_oracle_quantize_rows_static(const double* x, int64_t rows, int64_t cols, int bits,
                                    const double* s, const int32_t* z, uint8_t* codes) {
  /* quant.cpp:150-160 (frozen params) then 169-175 */
  if (!bits_supported(bits)) return 1;
  for (int64_t i = 0; i < rows * cols; ++i)
    if (!isfinite(x[i])) return 1;
  const double qmax = (double)((1 << bits) - 1);
  for (int64_t r = 0; r < rows; ++r) quantize_row(x + r * cols, cols, s[r], z[r], qmax, codes + r * cols);
  return 0;
}

void dtq_oracle_dequantize_rows(const uint8_t* codes, int64_t rows, int64_t cols,
                                const double* s, const int32_t* z, double* out) {
  /* quant.cpp:179-188 */
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      out[r * cols + c] = s[r] * ((int32_t)codes[r * cols + c] - z[r]);
}

static int is_pow2(int64_t n) { return n >= 2 && (n & (n - 1)) == 0; }

int dtq_oracle_fwht(double* d, int64_t n) {
  /* balance.cpp:22-33 */
  if (!is_pow2(n)) return 1;
  for (int64_t h = 1; h < n; h <<= 1)
    for (int64_t i = 0; i < n; i += h << 1)
      for (int64_t j = i; j < i + h; ++j) {
        const double a = d[j];
        const double b = d[j + h];
        d[j] = a + b;
        d[j + h] = a - b;
      }
  return 0;
}

/* std::mt19937_64 as fixed by the C++ standard ([rand.predef]):
 * w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29 d=0x5555555555555555
 * s=17 b=0x71d67fffeda60000 t=37 c=0xfff7eee000000000 l=43
 * f=6364136223846793005.  Default-seeded engine check: the 10000th
 * output is 9981545732273789042 (asserted in tests/test_oracle.py). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* e, uint64_t seed) {
  e->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    e->mt[i] = 6364136223846793005ULL * (e->mt[i - 1] ^ (e->mt[i - 1] >> 62)) + (uint64_t)i;
  e->idx = 312;
}

static uint64_t mt64_next(mt64_t* e) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (e->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (e->mt[i] & UM) | (e->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      e->mt[i] = e->mt[(i + 156) % 312] ^ xa;
    }
    e->idx = 0;
  }
  uint64_t y = e->mt[e->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= (y >> 43);
  return y;
}

uint64_t dtq_oracle_mt19937_64_nth(uint64_t seed, int64_t n) {
  mt64_t e;
  mt64_seed(&e, seed);
  uint64_t v = 0;
  for (int64_t i = 0; i < n; ++i) v = mt64_next(&e);
  return v;
}

void dtq_oracle_hadamard_signs(int64_t n, int randomize, uint64_t seed, int8_t* out) {
  /* balance.cpp:73-78 */
  if (!randomize) {
    for (int64_t i = 0; i < n; ++i) out[i] = 1;
    return;
  }
  mt64_t e;
  mt64_seed(&e, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = (mt64_next(&e) & 1ULL) ? (int8_t)1 : (int8_t)-1;
}

int dtq_oracle_rotate_blocks(double* x, int64_t rows, int64_t cols, int64_t hblock,
                             const int8_t* signs) {
  /* balance.cpp:94-107 applied per hblock-wide column block */
  if (!is_pow2(hblock) || cols % hblock != 0) return 1;
  const double norm = 1.0 / sqrt((double)hblock);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; j += hblock) {
      double* row = x + r * cols + j;
      for (int64_t c = 0; c < hblock; ++c) row[c] *= signs[j + c];
      dtq_oracle_fwht(row, hblock);
      for (int64_t c = 0; c < hblock; ++c) row[c] *= norm;
    }
  return 0;
}

int dtq_oracle_scaling_mask(const double* act_amax, const double* w_amax, int64_t n,
                            double alpha, double* s_out) {
  /* balance.cpp:35-55 */
  if (alpha < 0.0 || alpha > 1.0) return 1;
  for (int64_t i = 0; i < n; ++i) {
    const double a = act_amax[i], w = w_amax[i];
    if (a <= 0.0 || w <= 0.0 || !isfinite(a) || !isfinite(w)) {
      s_out[i] = 1.0;
      continue;
    }
    const double s = pow(a, alpha) / pow(w, 1.0 - alpha);
    s_out[i] = clampd(s, 1e-5, 1e5);
  }
  return 0;
}

void dtq_oracle_scale_x(double* x, int64_t rows, int64_t cols, const double* s) {
  /* balance.cpp:62-63 */
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) x[r * cols + c] /= s[c];
}

void dtq_oracle_scale_w(double* w, int64_t rows, int64_t cols, const double* s) {
  /* balance.cpp:64-65 */
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) w[r * cols + c] *= s[c];
}

void dtq_oracle_modulate(double* x, int64_t rows, int64_t cols, const double* scale,
                         const double* shift) {
  /* toydit.cpp:366-368 */
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c)
      x[r * cols + c] = x[r * cols + c] * (1.0 + scale[c]) + shift[c];
}

void dtq_oracle_gelu(double* x, int64_t n) {
  /* toydit.cpp:83 */
  const double sqrt2 = 1.4142135623730951;
  for (int64_t i = 0; i < n; ++i) x[i] = 0.5 * x[i] * (1.0 + erf(x[i] / sqrt2));
}

void dtq_oracle_layernorm(double* x, int64_t rows, int64_t cols, double eps) {
  /* no reference counterpart; torch.nn.functional.layer_norm semantics:
   * mean, biased variance of the centred values, (x - mean) / sqrt(var + eps) */
  for (int64_t r = 0; r < rows; ++r) {
    double* v = x + r * cols;
    double mean = 0.0, var = 0.0;
    for (int64_t c = 0; c < cols; ++c) mean += v[c];
    mean /= (double)cols;
    for (int64_t c = 0; c < cols; ++c) var += (v[c] - mean) * (v[c] - mean);
    var /= (double)cols;
    const double inv = 1.0 / sqrt(var + eps);
    for (int64_t c = 0; c < cols; ++c) v[c] = (v[c] - mean) * inv;
  }
}

int dtq_oracle_overflow_guard(int act_bits, int weight_bits, int64_t c_in) {
  /* qgemm.cpp:29-34 */
  const int64_t max_term = (int64_t)((1 << act_bits) - 1) * ((int64_t)1 << (weight_bits - 1));
  if (c_in <= 0) return 1;
  return (max_term > INT64_MAX / c_in) ? 2 : 0;
}

typedef struct {
  const uint8_t* xc;
  const int32_t* zx;
  const int32_t* wsym;
  const int64_t* wsum;
  int64_t K, N, r0, r1;
  int64_t* acc;
} acc_job_t;

static void* acc_rows(void* arg) {
  /* qgemm.cpp:52-60 on rows [r0, r1) */
  const acc_job_t* j = (const acc_job_t*)arg;
  for (int64_t t = j->r0; t < j->r1; ++t) {
    const uint8_t* xi = j->xc + t * j->K;
    for (int64_t o = 0; o < j->N; ++o) {
      const int32_t* wo = j->wsym + o * j->K;
      int64_t a = 0;
      for (int64_t c = 0; c < j->K; ++c) a += (int64_t)xi[c] * wo[c];
      a -= (int64_t)j->zx[t] * j->wsum[o];
      j->acc[t * j->N + o] = a;
    }
  }
  return NULL;
}

int dtq_oracle_num_cpus(void) {
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

int dtq_oracle_qlinear_acc(const uint8_t* xc, const int32_t* zx, int64_t M, int64_t K,
                           const uint8_t* wc, const int32_t* zw, int64_t N, int64_t* acc,
                           int threads) {
  /* qgemm.cpp:40-49: w_sym = code - z_w, row sums; 52-60: int64 dot + correction.
   * Rows are independent, so they are split over `threads` pthreads. */
  int32_t* wsym = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N * K));
  int64_t* wsum = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  if (!wsym || !wsum) {
    free(wsym);
    free(wsum);
    return 1;
  }
  for (int64_t o = 0; o < N; ++o) {
    int64_t sum = 0;
    for (int64_t c = 0; c < K; ++c) {
      const int32_t v = (int32_t)wc[o * K + c] - zw[o];
      wsym[o * K + c] = v;
      sum += v;
    }
    wsum[o] = sum;
  }
  if (threads <= 0) threads = dtq_oracle_num_cpus();
  if (threads > 256) threads = 256;
  if ((int64_t)threads > M) threads = (int)(M > 0 ? M : 1);
  pthread_t tid[256];
  acc_job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (acc_job_t){xc, zx, wsym, wsum, K, N, M * t / threads, M * (t + 1) / threads, acc};
  }
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, acc_rows, &jobs[t]);
  acc_rows(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  free(wsym);
  free(wsum);
  return 0;
}

void dtq_oracle_qlinear_epilogue(const int64_t* acc, const double* sx, int64_t M,
                                 const double* sw, const double* bias, int64_t N,
                                 double* y) {
  /* qgemm.cpp:61-63: out = s_x * s_w * (double)acc; out += bias */
  for (int64_t t = 0; t < M; ++t)
    for (int64_t o = 0; o < N; ++o) {
      double out = sx[t] * sw[o] * (double)acc[t * N + o];
      if (bias) out += bias[o];
      y[t * N + o] = out;
    }
}

int dtq_oracle_qlinear_forward(const double* x, int64_t M, int64_t K, int act_bits,
                               const uint8_t* wc, const double* sw, const int32_t* zw,
                               int weight_bits, int64_t N, const double* bias, double* y,
                               int threads) {
  /* qgemm.cpp:23-67 */
  const int g = dtq_oracle_overflow_guard(act_bits, weight_bits, K);
  if (g) return g;
  uint8_t* xc = (uint8_t*)malloc((size_t)(M * K));
  double* sx = (double*)malloc(sizeof(double) * (size_t)M);
  int32_t* zx = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  int64_t* acc = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M * N));
  int st = 1;
  if (xc && sx && zx && acc) {
    st = dtq_oracle_quantize_rows(x, M, K, act_bits, 0, xc, sx, zx);
    if (!st) st = dtq_oracle_qlinear_acc(xc, zx, M, K, wc, zw, N, acc, threads);
    if (!st) dtq_oracle_qlinear_epilogue(acc, sx, M, sw, bias, N, y);
  }
  free(xc);
  free(sx);
  free(zx);
  free(acc);
  return st;
}

int64_t dtq_oracle_pack_codes(const uint8_t* codes, int64_t count, int bits, uint8_t* out) {
  /* trace_io.cpp:79-91 */
  if (!bits_supported(bits)) return -1;
  const int64_t nbytes = (count * bits + 7) / 8;
  memset(out, 0, (size_t)nbytes);
  int64_t bitpos = 0;
  for (int64_t i = 0; i < count; ++i) {
    const uint8_t code = codes[i];
    if (code >= (1u << bits)) return -1;
    out[bitpos / 8] |= (uint8_t)(code << (bitpos % 8));
    if (bitpos % 8 + bits > 8) out[bitpos / 8 + 1] |= (uint8_t)(code >> (8 - bitpos % 8));
    bitpos += bits;
  }
  return nbytes;
}

int dtq_oracle_unpack_codes(const uint8_t* bytes, int64_t nbytes, int bits, int64_t count,
                            uint8_t* out) {
  /* trace_io.cpp:93-109 */
  if (!bits_supported(bits)) return 1;
  if (nbytes != (count * bits + 7) / 8) return 1;
  const uint8_t mask = (uint8_t)((1u << bits) - 1);
  int64_t bitpos = 0;
  for (int64_t i = 0; i < count; ++i) {
    uint16_t v = (uint16_t)(bytes[bitpos / 8] >> (bitpos % 8));
    if (bitpos % 8 + bits > 8 && bitpos / 8 + 1 < nbytes)
      v |= (uint16_t)((uint16_t)bytes[bitpos / 8 + 1] << (8 - bitpos % 8));
    out[i] = (uint8_t)(v & mask);
    bitpos += bits;
  }
  return 0;
}
