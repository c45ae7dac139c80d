// parity_kernels.cu -- fp64 device kernels for the reference operations that
// are not on the timed path (static quantize for every grouping, dequantize,
// apply_scaling / rotate_channels, the fp64 float-path GEMM).  Each keeps
// the reference's operation order so results are bit-identical; they back
// the C++ drop-in (include/dtq) and the parity tests.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/dtq_capi.h"

namespace {

int last_cuda(const char* what);

__device__ __forceinline__ int64_t group_of(int grouping, int64_t gs, int64_t r, int64_t c,
                                            int64_t cols) {
  // quant.cpp:36-45
  switch (grouping) {
    case 0: return 0;
    case 1:
    case 3: return r;
    case 2: return c;
    default: return r * (cols / gs) + c / gs;
  }
}

__global__ void quantize_static_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                       int64_t ldx, double qmax, int grouping, int64_t gs,
                                       const double* __restrict__ s, const int32_t* __restrict__ z,
                                       uint8_t* __restrict__ codes, int64_t ldc) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t g = group_of(grouping, gs, r, c, cols);
    // quant.cpp:171-173: k = round_even(x / s) + z, clamped, cast
    const double k = rint(x[r * ldx + c] / s[g]) + static_cast<double>(z[g]);
    codes[r * ldc + c] = static_cast<uint8_t>(fmin(fmax(k, 0.0), qmax));
  }
}

__global__ void dequantize_kernel(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols,
                                  int64_t ldc, int grouping, int64_t gs,
                                  const double* __restrict__ s, const int32_t* __restrict__ z,
                                  double* __restrict__ out, int64_t ldo) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t g = group_of(grouping, gs, r, c, cols);
    out[r * ldo + c] = s[g] * static_cast<double>(static_cast<int32_t>(codes[r * ldc + c]) - z[g]);
  }
}

// One CTA per (row, hblock-wide block): scale, signs, in-smem FWHT with the
// reference butterfly order (balance.cpp:22-33), normalise.
// raw_fwht: the butterflies alone (fwht, balance.cpp:22-33), no signs / norm.
__global__ void balance_kernel(const double* x, int64_t cols, int64_t ldx,
                               const double* __restrict__ smooth, int smooth_mul,
                               const int8_t* __restrict__ signs, int64_t hb, double* out,
                               int64_t ldo, int raw_fwht = 0) {
  extern __shared__ double buf[];
  const int64_t r = blockIdx.y;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * hb;
  for (int64_t c = threadIdx.x; c < hb; c += blockDim.x) {
    double v = x[r * ldx + base + c];
    if (smooth) v = smooth_mul ? v * smooth[base + c] : v / smooth[base + c];
    if (signs) v *= static_cast<double>(signs[base + c]);
    buf[c] = v;
  }
  __syncthreads();
  if (signs || raw_fwht) {
    for (int64_t h = 1; h < hb; h <<= 1) {
      for (int64_t p = threadIdx.x; p < hb / 2; p += blockDim.x) {
        const int64_t j = (p / h) * (2 * h) + (p % h);
        const double a = buf[j], b = buf[j + h];
        buf[j] = a + b;
        buf[j + h] = a - b;
      }
      __syncthreads();
    }
  }
  const double norm = signs ? 1.0 / sqrt(static_cast<double>(hb)) : 1.0;
  for (int64_t c = threadIdx.x; c < hb; c += blockDim.x)
    out[r * ldo + base + c] = signs ? buf[c] * norm : buf[c];
}

__global__ void matmul_nt_f64_kernel(const double* __restrict__ x, int64_t M, int64_t K,
                                     const double* __restrict__ w, int64_t N,
                                     const double* __restrict__ bias, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < M * N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, o = i % N;
    double acc = 0.0;
    for (int64_t k = 0; k < K; ++k) acc = __dadd_rn(acc, __dmul_rn(x[t * K + k], w[o * K + k]));
    if (bias) acc = __dadd_rn(acc, bias[o]);  // qgemm.cpp:74-76 adds bias after the GEMM
    y[i] = acc;
  }
}

// Dynamic per-row params for rows wider than the row quantizer's tile
// (the drop-in's per_tensor() over a whole matrix, per_channel() with many
// rows): per-chunk fp64 min / max (exact operations, so any split gives the
// reference's values), then one thread per row derives s, z exactly as
// compute_minmax_params / compute_symmetric_params (quant.cpp:90-124).
__global__ void wide_minmax_kernel(const double* __restrict__ x, int64_t cols, int64_t ldx,
                                   int64_t chunk, double2* __restrict__ part,
                                   int32_t* __restrict__ status) {
  const int64_t r = blockIdx.y;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * chunk;
  const int64_t c1 = c0 + chunk < cols ? c0 + chunk : cols;
  double mn = __longlong_as_double(0x7ff0000000000000LL), mx = -mn;
  bool bad = false;
  for (int64_t c = c0 + threadIdx.x; c < c1; c += blockDim.x) {
    const double v = x[r * ldx + c];
    bad |= !isfinite(v);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  __shared__ double smn[32], smx[32];
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = 0;
  for (int o = 16; o >= 1; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __syncthreads();
  if (bad) sbad = 1;
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      mn = fmin(mn, smn[w]);
      mx = fmax(mx, smx[w]);
    }
    part[r * gridDim.x + blockIdx.x] = make_double2(mn, mx);
    if (sbad && status) atomicOr(status, 1);
  }
}

__global__ void wide_params_kernel(const double2* __restrict__ part, int64_t rows, int nchunks,
                                   int bits, int symmetric, double* __restrict__ scale,
                                   int32_t* __restrict__ zero) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  double mn = part[r * nchunks].x, mx = part[r * nchunks].y;
  for (int i = 1; i < nchunks; ++i) {
    mn = fmin(mn, part[r * nchunks + i].x);
    mx = fmax(mx, part[r * nchunks + i].y);
  }
  const double qmax = static_cast<double>((1 << bits) - 1);
  double s, z;
  if (symmetric) {  // quant.cpp:115-124
    const double amax = fmax(fabs(mn), fabs(mx));
    z = static_cast<double>(1 << (bits - 1));
    s = amax > 0.0 ? amax / static_cast<double>((1 << (bits - 1)) - 1) : 1.0;
  } else if (mx == mn) {  // quant.cpp:90-113, degenerate group
    s = 1.0;
    z = fmin(fmax(rint(-mn), 0.0), qmax);
  } else {
    const double lo = (0.0 < mn) ? 0.0 : mn;
    const double hi = (mx < 0.0) ? 0.0 : mx;
    s = (hi - lo) / qmax;
    z = fmin(fmax(rint(-lo / s), 0.0), qmax);
  }
  scale[r] = s;
  zero[r] = static_cast<int32_t>(z);
}

// col_absmax / row_absmax (matrix.hpp:95-109): max |x| per column / row in
// fp64 -- max is exact, so any reduction order gives the reference's values
// (fmax drops NaN like the reference's std::max(acc, |x|) with acc first).
__global__ void col_absmax_kernel(const double* __restrict__ x, int64_t rows, int64_t cols,
                                  int64_t ldx, int64_t rows_per, double* __restrict__ part) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per;
  const int64_t r1 = r0 + rows_per < rows ? r0 + rows_per : rows;
  double m = 0.0;
  for (int64_t r = r0; r < r1; ++r) m = fmax(m, fabs(x[r * ldx + c]));  // coalesced over c
  part[blockIdx.y * cols + c] = m;
}

__global__ void max_fold_kernel(const double* __restrict__ part, int64_t n, int nparts,
                                double* __restrict__ out) {
  const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (c >= n) return;
  double m = 0.0;
  for (int i = 0; i < nparts; ++i) m = fmax(m, part[i * n + c]);
  out[c] = m;
}

__global__ void row_absmax_kernel(const double* __restrict__ x, int64_t cols, int64_t ldx,
                                  double* __restrict__ out) {
  const int64_t r = blockIdx.x;
  double m = 0.0;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) m = fmax(m, fabs(x[r * ldx + c]));
  for (int o = 16; o >= 1; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    out[r] = m;
  }
}

int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 148 * 32 ? (g > 0 ? g : 1) : 148 * 32);
}

}  // namespace

extern "C" {

int dtq_quantize_static(const double* x, int64_t rows, int64_t cols, int64_t ldx, int bits,
                        int grouping, int64_t group_size, const double* scale,
                        const int32_t* zero, uint8_t* codes, int64_t ldc, void* stream) {
  if (rows <= 0 || cols <= 0 || !x || !scale || !zero || !codes) return DTQ_ERR_INVALID_ARGUMENT;
  if (!(bits == 2 || bits == 4 || bits == 6 || bits == 8)) return DTQ_ERR_INVALID_ARGUMENT;
  if (grouping == 4 && (group_size <= 0 || cols % group_size)) return DTQ_ERR_INVALID_ARGUMENT;
  quantize_static_kernel<<<grid_for(rows * cols), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, rows, cols, ldx, static_cast<double>((1 << bits) - 1), grouping, group_size, scale, zero,
      codes, ldc);
  return last_cuda("quantize_static");
}

int dtq_dequantize(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ldc, int grouping,
                   int64_t group_size, const double* scale, const int32_t* zero, double* out,
                   int64_t ldo, void* stream) {
  if (rows <= 0 || cols <= 0 || !codes || !scale || !zero || !out) return DTQ_ERR_INVALID_ARGUMENT;
  if (grouping == 4 && (group_size <= 0 || cols % group_size)) return DTQ_ERR_INVALID_ARGUMENT;
  dequantize_kernel<<<grid_for(rows * cols), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      codes, rows, cols, ldc, grouping, group_size, scale, zero, out, ldo);
  return last_cuda("dequantize");
}

int dtq_balance_apply(const double* x, int64_t rows, int64_t cols, int64_t ldx,
                      const double* smooth, int smooth_mul, const int8_t* signs, int64_t hblock,
                      double* out, int64_t ldo, void* stream) {
  if (rows <= 0 || cols <= 0 || !x || !out) return DTQ_ERR_INVALID_ARGUMENT;
  const int64_t hb = signs ? hblock : (cols < 1024 ? cols : 1024);
  if (signs && (hb < 2 || (hb & (hb - 1)) != 0 || cols % hb != 0 || hb > 16384))
    return DTQ_ERR_INVALID_ARGUMENT;
  if (!signs && cols % hb != 0) {
    // plain scaling with no rotation: any width, one "block" per row
    if (cols > 16384) return DTQ_ERR_INVALID_ARGUMENT;
    dim3 grid(1, static_cast<unsigned>(rows));
    balance_kernel<<<grid, 256, cols * sizeof(double), static_cast<cudaStream_t>(stream)>>>(
        x, cols, ldx, smooth, smooth_mul, nullptr, cols, out, ldo);
    return last_cuda("balance_apply");
  }
  dim3 grid(static_cast<unsigned>(cols / hb), static_cast<unsigned>(rows));
  const size_t smem = hb * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(balance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  balance_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      x, cols, ldx, smooth, smooth_mul, signs, hb, out, ldo);
  return last_cuda("balance_apply");
}

int dtq_col_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                       void* stream) {
  if (rows <= 0 || cols <= 0 || ldx < cols || !x || !out) return DTQ_ERR_INVALID_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // row slabs of 64 rows, each column's slab maxima folded in a second pass
  const int64_t rows_per = 64;
  const int64_t nparts = (rows + rows_per - 1) / rows_per;
  if (nparts > 65535) return DTQ_ERR_INVALID_ARGUMENT;
  double* part = nullptr;
  if (cudaMallocAsync(&part, nparts * cols * sizeof(double), st) != cudaSuccess)
    return DTQ_ERR_CUDA;
  dim3 grid(static_cast<unsigned>((cols + 127) / 128), static_cast<unsigned>(nparts));
  col_absmax_kernel<<<grid, 128, 0, st>>>(x, rows, cols, ldx, rows_per, part);
  max_fold_kernel<<<static_cast<unsigned>((cols + 127) / 128), 128, 0, st>>>(
      part, cols, static_cast<int>(nparts), out);
  cudaFreeAsync(part, st);
  return last_cuda("col_absmax");
}

int dtq_row_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, double* out,
                       void* stream) {
  if (rows <= 0 || cols <= 0 || ldx < cols || !x || !out) return DTQ_ERR_INVALID_ARGUMENT;
  if (rows > 0x7fffffff) return DTQ_ERR_INVALID_ARGUMENT;
  row_absmax_kernel<<<static_cast<unsigned>(rows), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, cols, ldx, out);
  return last_cuda("row_absmax");
}

int dtq_fwht_f64(double* x, int64_t rows, int64_t n, int64_t ldx, void* stream) {
  // fwht (balance.cpp:22-33) on each row, in place: the reference butterfly
  // order (a + b low, a - b high; h = 1, 2, 4, ...), unnormalised, no signs
  if (rows <= 0 || n <= 0 || (n & (n - 1)) != 0 || n > 16384 || ldx < n || !x)
    return DTQ_ERR_INVALID_ARGUMENT;
  if (n == 1) return DTQ_OK;
  dim3 grid(1, static_cast<unsigned>(rows));
  const size_t smem = n * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(balance_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  balance_kernel<<<grid, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      x, n, ldx, nullptr, 0, nullptr, n, x, ldx, /*raw_fwht=*/1);
  return last_cuda("fwht");
}

int dtq_matmul_nt_f64(const double* x, int64_t M, int64_t K, const double* w, int64_t N,
                      const double* bias, double* y, void* stream) {
  if (M <= 0 || K <= 0 || N <= 0 || !x || !w || !y) return DTQ_ERR_INVALID_ARGUMENT;
  matmul_nt_f64_kernel<<<grid_for(M * N), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, M, K, w, N, bias, y);
  return last_cuda("matmul_nt_f64");
}

}  // extern "C"

// fp64 rows of any width, exact mode, no prologue / balance (capi.cu routes
// rows wider than the tile quantizers here)
int dtq_quantize_rows_wide_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, int bits,
                               int symmetric, uint8_t* codes, int64_t ldc, double* scale,
                               int32_t* zero, int32_t* status, cudaStream_t st) {
  constexpr int64_t kChunk = 8192;
  const int64_t nchunks = (cols + kChunk - 1) / kChunk;
  if (nchunks > 65535 || rows > 65535) return DTQ_ERR_INVALID_ARGUMENT;
  double2* part = nullptr;
  if (cudaMallocAsync(&part, rows * nchunks * sizeof(double2), st) != cudaSuccess)
    return DTQ_ERR_CUDA;
  dim3 grid(static_cast<unsigned>(nchunks), static_cast<unsigned>(rows));
  wide_minmax_kernel<<<grid, 256, 0, st>>>(x, cols, ldx, kChunk, part, status);
  wide_params_kernel<<<static_cast<unsigned>((rows + 127) / 128), 128, 0, st>>>(
      part, rows, static_cast<int>(nchunks), bits, symmetric, scale, zero);
  quantize_static_kernel<<<grid_for(rows * cols), 256, 0, st>>>(
      x, rows, cols, ldx, static_cast<double>((1 << bits) - 1), 1, 0, scale, zero, codes, ldc);
  cudaFreeAsync(part, st);
  return last_cuda("quantize_rows_wide");
}

namespace {
int last_cuda(const char* what) {
  (void)what;
  return cudaGetLastError() == cudaSuccess ? DTQ_OK : DTQ_ERR_CUDA;
}
}  // namespace
