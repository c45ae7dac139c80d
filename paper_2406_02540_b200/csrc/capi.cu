// capi.cu -- implementation of include/dtq_capi.h on sm_100a.
//
// Host-side plumbing only: argument validation with the reference's error
// conventions, handle management (the prepared QuantLinear lives in HBM),
// TMA descriptor encoding, kernel selection and launch.  All arithmetic is
// in fused_quant.cuh (activation / weight quantizer) and qgemm_sm100.cuh
// (tcgen05 integer GEMM).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/dtq_capi.h"
#include "launch.h"

// parity_kernels.cu
int dtq_quantize_rows_wide_f64(const double* x, int64_t rows, int64_t cols, int64_t ldx, int bits,
                               int symmetric, uint8_t* codes, int64_t ldc, double* scale,
                               int32_t* zero, int32_t* status, cudaStream_t st);

namespace {

// NVTX range over a C-ABI call (header-only NVTX3: a few ns when no tool is
// attached; Nsight Systems / ncu --nvtx show the host calls around the
// kernels they launch)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(DTQ_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                  \
  } while (0)

#define DTQ_TRY(expr)          \
  do {                         \
    int st_ = (expr);          \
    if (st_ != DTQ_OK) return st_; \
  } while (0)

bool bits_supported(int b) { return b == 2 || b == 4 || b == 6 || b == 8; }

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct DeviceInfo {
  int dev = -1;
  int sms = 0;
  int major = 0;
};

// Per-thread cache of the current device's properties: one cudaGetDevice
// (a few tens of ns) per call instead of a device count + property query.
DeviceInfo& device_info() {
  thread_local DeviceInfo info;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    info.dev = -1;
    info.major = 0;
    return info;
  }
  if (info.dev != dev) {
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
      info.dev = dev;
      info.sms = p.multiProcessorCount;
      info.major = p.major;
    } else {
      info.dev = -1;
      info.major = 0;
    }
  }
  return info;
}

int check_device() {
  DeviceInfo& d = device_info();
  if (d.dev < 0) {
    cudaGetLastError();  // clear the sticky "no device" error of the probe
    return fail(DTQ_ERR_CUDA, "no CUDA device (the sm_100a path has no CPU fallback)");
  }
  if (d.major != 10)
    return fail(DTQ_ERR_CUDA, "device compute capability %d.x is not sm_100 (B200)", d.major);
  return DTQ_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000,
                                         cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D u8 tensor [rows, cols] with row pitch `ld` bytes, box {box_cols, box_rows}.
int make_tmap_u8(CUtensorMap* m, const void* base, int64_t rows, int64_t cols, int64_t ld,
                 int box_cols, int box_rows, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return fail(DTQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) % 16 != 0 || ld % 16 != 0)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "TMA operand needs 16-byte aligned base and pitch");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(DTQ_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return DTQ_OK;
}

// row flags: 128-row blocks a forward can publish (M <= 1M rows)
constexpr int kMaxFlagBlocks = 8192;

// rotation blocks: the fused quantizers take up to 256 columns; wider blocks
// (up to a full 16384-point rotation) take the fp64 pre-pass
constexpr int kMaxFusedHblock = 256;
constexpr int kMaxHblock = 16384;

// any input dtype -> dense fp64 (the pre-pass of wide rotation blocks);
// non-finite values set status like the fused quantizers
__global__ void to_f64_kernel(const void* __restrict__ x, int dt, int64_t rows, int64_t cols,
                              int64_t ldx, double* __restrict__ out, int32_t* status) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols, j = r * ldx + c;
    double v;
    switch (dt) {
      case DTQ_F16: v = static_cast<double>(__half2float(static_cast<const __half*>(x)[j])); break;
      case DTQ_BF16:
        v = static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(x)[j]));
        break;
      case DTQ_F32: v = static_cast<double>(static_cast<const float*>(x)[j]); break;
      default: v = static_cast<const double*>(x)[j]; break;
    }
    if (status && !isfinite(v)) atomicOr(status, 1);
    out[i] = v;
  }
}

// ------------------------------------------------------------------ FQ launch
// (kernel instantiations live in fq_kernels.cu / fq_fast_*.cu)
int fq_error(cudaError_t e) {
  if (e != cudaSuccess) return fail(DTQ_ERR_CUDA, "fused quantizer launch: %s", cudaGetErrorString(e));
  return DTQ_OK;
}

// fast-mode folded column multiplier: sign[c] / smooth[c] / sqrt(hblock)
__global__ void col_mul_kernel(const double* __restrict__ smooth, const int8_t* __restrict__ signs,
                               int hblock, int64_t K, float* __restrict__ out) {
  const double norm = signs ? 1.0 / sqrt(static_cast<double>(hblock)) : 1.0;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < K;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double m = norm;
    if (smooth) m /= smooth[c];
    if (signs && signs[c] < 0) m = -m;
    out[c] = static_cast<float>(m);
  }
}

size_t dtype_size(int dt) {
  switch (dt) {
    case DTQ_F16:
    case DTQ_BF16:
      return 2;
    case DTQ_F32:
    case DTQ_S32:
      return 4;
    case DTQ_F64:
      return 8;
  }
  return 0;
}

// diagnostics: per-warp phase cycle counters of the fast quantizer, only when
// DTQ_DEBUG_FQ_PROBE=1 (read back with dtq_diag_fq_probe_ptr)
unsigned long long* fq_probe_buffer() {
  static unsigned long long* p = [] {
    const char* e = std::getenv("DTQ_DEBUG_FQ_PROBE");
    unsigned long long* b = nullptr;
    if (e && e[0] == '1' && cudaMalloc(&b, 65536 * 8 * 8) == cudaSuccess)
      cudaMemset(b, 0, 65536 * 8 * 8);
    return b;
  }();
  return p;
}

// Row quantizer; `smooth_mul` selects W * s (weight side) instead of X / s.
int quantize_rows_impl(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                       int bits, int symmetric, int mode, int smooth_mul, const double* smooth_d,
                       const float* col_mul, const int8_t* signs, int hblock,
                       const dtq_prologue* pro, uint8_t* codes, int64_t ldc, double* scale,
                       int32_t* zero, int32_t* status, cudaStream_t st,
                       bool col_mul_const = true, uint32_t* ready = nullptr,
                       int partner_regs = 0, int partner_smem = 0, int* flags_used = nullptr,
                       const dtq_w4::Unpack* w4job = nullptr, int* w4_done = nullptr) {
  if (flags_used) *flags_used = 0;
  if (w4_done) *w4_done = 0;
  if (rows <= 0 || cols <= 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: empty matrix");
  if (!bits_supported(bits))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: bits must be one of {2,4,6,8}");
  if (ldx < cols || ldc < cols) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: pitch < cols");
  if (!x || !codes || !scale || !zero)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: null pointer");
  if (dtype_size(x_dtype) == 0 || x_dtype == DTQ_S32)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: bad input dtype %d", x_dtype);
  if (signs) {
    if (hblock < 8 || hblock > kMaxHblock || (hblock & (hblock - 1)) != 0)
      return fail(DTQ_ERR_INVALID_ARGUMENT,
                  "hadamard: block must be a power of two in [8, %d]", kMaxHblock);
    if (cols % hblock != 0)
      return fail(DTQ_ERR_INVALID_ARGUMENT, "rotate_channels: channel count %lld not a multiple "
                  "of the rotation block %d", (long long)cols, hblock);
  }
  const int kind = pro ? pro->kind : DTQ_PROLOGUE_NONE;
  if (signs && hblock > kMaxFusedHblock) {
    // rotation blocks wider than the fused kernels' (a reference checkpoint
    // stores weights rotated by the full C_in-point Hadamard, dtq_main.cpp
    // cmd_quantize): fp64 copy, apply_scaling + rotate_channels in the
    // reference order (balance_kernel, balance.cpp:57-67, 94-107), then the
    // exact quantizer on the balanced rows.  Always fp64 (never less exact).
    if (kind != DTQ_PROLOGUE_NONE)
      return fail(DTQ_ERR_UNSUPPORTED, "prologue with a rotation block wider than %d",
                  kMaxFusedHblock);
    DTQ_TRY(check_device());
    double* tmp = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tmp), rows * cols * sizeof(double), st));
    const int64_t n = rows * cols;
    to_f64_kernel<<<static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 32)), 256, 0, st>>>(
        x, x_dtype, rows, cols, ldx, tmp, status);
    int r = cudaGetLastError() == cudaSuccess ? DTQ_OK : fail(DTQ_ERR_CUDA, "to_f64 launch");
    if (r == DTQ_OK &&
        dtq_balance_apply(tmp, rows, cols, cols, smooth_d, smooth_mul, signs, hblock, tmp, cols,
                          st) != DTQ_OK)
      r = fail(DTQ_ERR_CUDA, "balance_apply launch failed");
    if (r == DTQ_OK)
      r = quantize_rows_impl(tmp, DTQ_F64, rows, cols, cols, bits, symmetric, DTQ_MODE_EXACT, 0,
                             nullptr, nullptr, nullptr, 0, nullptr, codes, ldc, scale, zero,
                             status, st);
    cudaFreeAsync(tmp, st);
    return r;
  }
  if (cols > 16384) {
    // wider groups (the drop-in's per_tensor() / per_channel() params):
    // chunked fp64 min / max, exact params, static codes
    if (!(mode == DTQ_MODE_EXACT || x_dtype == DTQ_F64) || x_dtype != DTQ_F64 || smooth_d ||
        signs || kind != DTQ_PROLOGUE_NONE || smooth_mul)
      return fail(DTQ_ERR_INVALID_ARGUMENT,
                  "quantize: rows wider than 16384 need fp64 input, exact mode, no balance "
                  "or prologue");
    DTQ_TRY(check_device());
    const int r = dtq_quantize_rows_wide_f64(static_cast<const double*>(x), rows, cols, ldx, bits,
                                             symmetric, codes, ldc, scale, zero, status, st);
    if (r != DTQ_OK) return fail(r, "quantize: wide-row launch failed");
    return DTQ_OK;
  }
  if (kind < 0 || kind > 3) return fail(DTQ_ERR_INVALID_ARGUMENT, "bad prologue kind");
  if ((kind == DTQ_PROLOGUE_MODULATE || kind == DTQ_PROLOGUE_LN_MODULATE) &&
      (!pro->scale || !pro->shift))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "modulate prologue needs scale and shift");
  DTQ_TRY(check_device());

  const bool exact = mode == DTQ_MODE_EXACT || x_dtype == DTQ_F64;
  if (!exact && smooth_mul)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "weight-side smoothing runs in exact mode only");
  if (!exact && (smooth_d || signs) && !col_mul)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "fast mode needs the folded column multiplier");
  const int64_t chunks = (cols + 7) / 8;
  const size_t es = dtype_size(x_dtype);
  const bool vec = cols % 8 == 0 && (ldx * es) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(x) % 16 == 0 && ldc % 8 == 0 &&
                   reinterpret_cast<uintptr_t>(codes) % 8 == 0 &&
                   (!smooth_d || reinterpret_cast<uintptr_t>(smooth_d) % 16 == 0) &&
                   (kind == 0 || kind == 2 ||
                    (reinterpret_cast<uintptr_t>(pro->scale) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(pro->shift) % 16 == 0));

  dtq_fq::FqArgs a{};
  a.x = x;
  a.M = rows;
  a.K = cols;
  a.ldx = ldx;
  a.codes = codes;
  a.ldc = ldc;
  a.scale = scale;
  a.zero = zero;
  a.bits = bits;
  a.symmetric = symmetric;
  a.smooth_d = exact ? smooth_d : nullptr;
  a.col_mul = exact ? nullptr : col_mul;
  a.col_mul_const = col_mul_const ? 1 : 0;
  a.signs = signs;
  a.hblock = signs ? hblock : 0;
  a.pro_scale = pro ? pro->scale : nullptr;
  a.pro_shift = pro ? pro->shift : nullptr;
  a.eps = pro ? pro->eps : 0.f;
  a.status = status;
  a.pro = kind;
  a.smooth_mul = smooth_mul;
  a.probe = fq_probe_buffer();
  static const int fq_dbg = [] {
    const char* e = std::getenv("DTQ_DEBUG_FQ");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = fq_dbg;
  const int sms = device_info().sms;

  // the fp32 kernel needs 16-byte rows, K % 128 == 0 and a 128-column
  // rotation block; anything else runs on the fp64 kernel (more precise,
  // never less exact)
  const bool fast = !exact && vec && cols % 128 == 0 && (!signs || hblock == 128);
  if (!fast) {
    if (!exact && (smooth_d || signs) && !smooth_d && !signs) return DTQ_ERR_INVALID_ARGUMENT;
    // CTA per row; 8-element chunks, 1 (K <= 8192) or 8 chunks per thread
    const int cpt = chunks <= 1024 ? 1 : 8;
    const int64_t align = signs ? (hblock / 8 > 16 ? hblock / 8 : 16) : 16;
    const int64_t tpr = round_up((chunks + cpt - 1) / cpt, align);
    if (tpr > (cpt == 1 ? 1024 : 256))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: cols too large");
    a.tpr = static_cast<int>(tpr);
    a.col_mul = nullptr;
    if (!exact) {
      // fp32 request on an unaligned / non-128-block input: exact kernel with
      // the fp64 transforms it needs
      if (smooth_d == nullptr && col_mul != nullptr && !signs)
        return fail(DTQ_ERR_UNSUPPORTED, "unaligned fast-mode input needs the fp64 smoothing vector");
      a.smooth_d = smooth_d;
    }
    return fq_error(dtq_launch_fq_exact(a, x_dtype, cpt, vec,
                                        static_cast<int>(round_up(tpr, 32)), sms, st));
  }
  // fast, register-resident tile kernel: one thread per (row, 128-column
  // block); needs 16-byte code rows for its bulk stores
  static const bool tile_off = [] {
    const char* e = std::getenv("DTQ_FQ_TILE");
    return e != nullptr && e[0] == '0';
  }();
  if (!tile_off && cols <= 8192 && ldc % 16 == 0 && reinterpret_cast<uintptr_t>(codes) % 16 == 0) {
    const bool has_b = kind == DTQ_PROLOGUE_MODULATE || kind == DTQ_PROLOGUE_LN_MODULATE;
    const bool has_a = has_b || col_mul != nullptr;
    const bool exact_v = kind == DTQ_PROLOGUE_NONE && !has_a && signs == nullptr;
    const int R = dtq_fq_tile_rows(rows, cols, static_cast<int>(es), has_a, has_b, kind, exact_v,
                                   sms);
    if (R > 0) {
      // row flags: the launcher keeps them only if the quantizer fits beside
      // the GEMM on every SM (and says so in *flags_used)
      a.ready = ready;
      a.partner_regs = partner_regs;
      a.partner_smem = partner_smem;
      a.flags_used = flags_used;
      if (w4job) a.w4 = *w4job;  // the tile kernel also expands a W4A8 forward's weights
      a.w4_done = w4_done;
      return fq_error(dtq_launch_fq_tile(a, static_cast<int>(es), x_dtype == DTQ_BF16 ? 1 : 0,
                                         signs != nullptr, R, sms, st));
    }
  }
  // fast: G 8-lane groups per row, R = 4/G rows per warp with R*K <= 4608
  // (18 KB fp32 park buffer per warp); warps per CTA sized for ~2 CTAs/SM
  int G = 2;
  while (G < 4 && (4 / G) * cols > 2304) G *= 2;
  static const int forced_g = [] {
    const char* e = std::getenv("DTQ_FQ_G");
    return e ? std::atoi(e) : 0;
  }();
  if (forced_g == 1 || forced_g == 2 || forced_g == 4) G = forced_g;
  const size_t wbytes = dtq_fq::fq_fast_warp_bytes(cols, G, static_cast<int>(es));
  int wpc = static_cast<int>((113 * 1024) / wbytes);
  wpc = wpc < 1 ? 1 : (wpc > 8 ? 8 : wpc);
  if (wbytes * wpc > 227 * 1024) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: cols too large");
  const int block = 32 * wpc;
  a.tpr = 32;
  const int cpt = G;
  const bool rot = signs != nullptr;
  switch (x_dtype) {
    case DTQ_F16: return fq_error(dtq_launch_fq_fast_f16(a, cpt, rot, block, sms, st));
    case DTQ_BF16: return fq_error(dtq_launch_fq_fast_bf16(a, cpt, rot, block, sms, st));
    default: return fq_error(dtq_launch_fq_fast_f32(a, cpt, rot, block, sms, st));
  }
}

// ------------------------------------------------------------------ weight prep kernels
// reference codes (z = 2^(b-1)) -> s8 w_sym rows (W8) or packed nibbles (W4),
// plus w_row_sum (qgemm.cpp:40-49).  One CTA per output channel.
__global__ void weight_pack_kernel(const uint8_t* __restrict__ codes, int64_t ldc, int64_t N,
                                   int64_t K, int wbits, int8_t* __restrict__ w8, int64_t ld8,
                                   uint8_t* __restrict__ w4, int64_t ld4,
                                   int32_t* __restrict__ wsum) {
  const int64_t o = blockIdx.x;
  if (o >= N) return;
  const int32_t z = 1 << (wbits - 1);
  int32_t sum = 0;
  if (wbits != 4) {  // 2-, 6- and 8-bit weights are stored as s8 w_sym
    for (int64_t c = threadIdx.x; c < ld8; c += blockDim.x) {
      int32_t v = 0;
      if (c < K) v = static_cast<int32_t>(codes[o * ldc + c]) - z;
      w8[o * ld8 + c] = static_cast<int8_t>(v);
      sum += v;
    }
  } else {
    // GEMM nibble layout (not the reference's stream order): each 32-bit word
    // holds columns 8i..8i+7 as signed nibbles n = c ^ 8 (= c - 8 in 4-bit
    // two's complement), byte k = n[8i+k] | n[8i+k+4] << 4, so the GEMM's
    // unpack to 16*(c-8) as s8 is two masks and a shift (w4_word_to_s8x8_x16)
    for (int64_t b = threadIdx.x; b < ld4; b += blockDim.x) {
      const int64_t c0 = 8 * (b >> 2) + (b & 3), c1 = c0 + 4;
      const uint32_t lo = c0 < K ? codes[o * ldc + c0] : 8u;  // pad: code 8 -> w_sym 0
      const uint32_t hi = c1 < K ? codes[o * ldc + c1] : 8u;
      w4[o * ld4 + b] = static_cast<uint8_t>((lo ^ 8u) | ((hi ^ 8u) << 4));
      sum += static_cast<int32_t>(lo) - 8 + static_cast<int32_t>(hi) - 8;
    }
  }
  __shared__ int32_t red[32];
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int i = 0; i < (blockDim.x + 31) / 32; ++i) s += red[i];
    wsum[o] = s;
  }
}

// trace_io LSB-first bit stream -> one code per byte (unpack_codes, trace_io.cpp:93-109)
__global__ void unpack_stream_kernel(const uint8_t* __restrict__ bytes, int64_t count, int bits,
                                     int64_t N, int64_t K, uint8_t* __restrict__ out,
                                     int64_t ldo) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t bitpos = i * bits;
    uint32_t v = bytes[bitpos / 8] >> (bitpos % 8);
    if (bitpos % 8 + bits > 8) v |= static_cast<uint32_t>(bytes[bitpos / 8 + 1]) << (8 - bitpos % 8);
    out[(i / K) * ldo + (i % K)] = static_cast<uint8_t>(v & ((1u << bits) - 1));
  }
}

__global__ void export_codes_kernel(const int8_t* __restrict__ w8, int64_t ld8,
                                    const uint8_t* __restrict__ w4, int64_t ld4, int wbits,
                                    int64_t N, int64_t K, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N * K;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t o = i / K, c = i % K;
    if (wbits != 4)
      out[i] = static_cast<uint8_t>(static_cast<int32_t>(w8[o * ld8 + c]) + (1 << (wbits - 1)));
    else  // the GEMM nibble layout of weight_pack_kernel
      out[i] = ((w4[o * ld4 + 4 * (c >> 3) + (c & 3)] >> ((c & 4) ? 4 : 0)) & 0xF) ^ 8;
  }
}

// fp64 parity epilogue (qgemm.cpp:61-63 operation order):
//   y = s_x[t] * s_w[o] * (double)acc + bias[o]
__global__ void parity_epilogue_kernel(const int32_t* __restrict__ acc, int64_t M, int64_t N,
                                       const double* __restrict__ s_x,
                                       const double* __restrict__ s_w,
                                       const double* __restrict__ bias, double* __restrict__ y,
                                       int64_t ldy) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, o = i % N;
    // explicit roundings: no FMA contraction, same as the reference's x86 build
    double out = __dmul_rn(__dmul_rn(s_x[t], s_w[o]), static_cast<double>(acc[i]));
    if (bias) out = __dadd_rn(out, bias[o]);
    y[t * ldy + o] = out;
  }
}

// W4A8 forward: the s8 weight expansion as its own kernel (w4_unpack.cuh),
// for quantizer kernels other than the tile kernel.  Launched
// programmatically after the quantizer: griddepcontrol.wait precedes every
// store (the previous forward's GEMM reads the same workspace until the
// quantizer, which waited for it, has completed).
__global__ void __launch_bounds__(256) w4_unpack_kernel(const dtq_w4::Unpack u) {
  dtq_ptx::pdl_wait();
  dtq_ptx::pdl_launch_dependents();
  dtq_w4::unpack_range(u, blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x,
                       static_cast<int64_t>(gridDim.x) * blockDim.x);
}

__global__ void to_f32_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t n,
                              int reciprocal) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<float>(reciprocal ? 1.0 / in[i] : in[i]);
}

}  // namespace

// ------------------------------------------------------------------ handle
struct dtq_qlinear_s {
  int64_t N = 0, K = 0;
  int wbits = 8, abits = 8;
  int8_t* w8 = nullptr;   // [N, ld8] s8 (W8)
  int64_t ld8 = 0;
  uint8_t* w4 = nullptr;  // [N, ld4] packed signed nibbles, GEMM order (W4; weight_pack_kernel)
  int64_t ld4 = 0;
  double* s_w = nullptr;      // [N]
  float* s_w_f = nullptr;     // [N]
  int32_t* wsum = nullptr;    // [N]
  double* bias = nullptr;     // [N] or null
  float* bias_f = nullptr;    // [N] or null
  double* smooth = nullptr;   // [K] or null
  float* col_mul = nullptr;     // [K] fast-mode folded sign / smooth / norm, or null
  int8_t* signs = nullptr;    // [K] or null
  int hblock = 0;
  CUtensorMap tmB[3];  // B operand boxes of 256, 128 and 64 rows
  // handle-owned scratch (forward without workspace, F64 output, host forward)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int32_t* acc32 = nullptr;
  size_t acc32_bytes = 0;
  void* hx = nullptr;
  size_t hx_bytes = 0;
  void* hy = nullptr;
  size_t hy_bytes = 0;
  int32_t* status = nullptr;
  // host-forward pipeline over row chunks: one stream per role (H2D copies,
  // quantize + GEMM, D2H copies) chained per chunk by events, so the copy
  // engines in the two directions never wait on each other's queue
  cudaStream_t ps[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t pe[2] = {nullptr, nullptr};          // fork / join
  std::vector<cudaEvent_t> ev_in, ev_out;          // per chunk: H2D done, GEMM done
  void* pws = nullptr;
  size_t pws_bytes = 0;
  std::mutex host_mu;  // forward_host is synchronous: one call per handle at a time
  // encoded A / Y tensor maps of recent calls (a layer sees the same few
  // activation / output buffers every step): encoding one costs ~1-2 us of
  // host time, more than a C2-sized quantizer launch
  struct TmapEntry {
    const void* base = nullptr;
    int64_t rows = 0, cols = 0, ld = 0;
    int box_cols = 0, box_rows = 0, swz = 0;
    CUtensorMap map;
  };
  static constexpr int kTmapCache = 16;
  TmapEntry tmaps[kTmapCache];
  int tmap_next = 0;
  std::mutex tmap_mu;
};

namespace {

// (zero_on: a forward workspace -- its row-flag counters must start at zero;
// zeroed stream-ordered on that stream)
int grow(void** p, size_t* cur, size_t need, cudaStream_t zero_on = nullptr,
         bool zero = false) {
  if (*cur >= need) return DTQ_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cur = 0;
  CUDA_TRY(cudaMalloc(p, need));
  *cur = need;
  if (zero) CUDA_TRY(cudaMemsetAsync(*p, 0, need, zero_on));
  return DTQ_OK;
}

void free_handle(dtq_qlinear_s* h) {
  void* ptrs[] = {h->w8, h->w4, h->s_w, h->s_w_f, h->wsum, h->bias, h->bias_f, h->smooth,
                  h->col_mul, h->signs, h->scratch, h->acc32, h->hx, h->hy, h->status};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h->pws) cudaFree(h->pws);
  for (cudaStream_t s : h->ps)
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : h->pe)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : h->ev_out) cudaEventDestroy(e);
  delete h;
}

// make_tmap_u8 through the handle's cache of recently encoded maps
int cached_tmap_u8(dtq_qlinear_s* h, CUtensorMap* m, const void* base, int64_t rows, int64_t cols,
                   int64_t ld, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
  std::lock_guard<std::mutex> lock(h->tmap_mu);
  for (const auto& e : h->tmaps) {
    if (e.base == base && e.rows == rows && e.cols == cols && e.ld == ld &&
        e.box_cols == box_cols && e.box_rows == box_rows && e.swz == static_cast<int>(swz)) {
      *m = e.map;
      return DTQ_OK;
    }
  }
  DTQ_TRY(make_tmap_u8(m, base, rows, cols, ld, box_cols, box_rows, swz));
  auto& e = h->tmaps[h->tmap_next];
  h->tmap_next = (h->tmap_next + 1) % dtq_qlinear_s::kTmapCache;
  e.base = base;
  e.rows = rows;
  e.cols = cols;
  e.ld = ld;
  e.box_cols = box_cols;
  e.box_rows = box_rows;
  e.swz = static_cast<int>(swz);
  e.map = *m;
  return DTQ_OK;
}

int alloc_status(dtq_qlinear_s* h, cudaStream_t st) {
  CUDA_TRY(cudaMalloc(&h->status, sizeof(int32_t)));
  CUDA_TRY(cudaMemsetAsync(h->status, 0, sizeof(int32_t), st));
  return DTQ_OK;
}

int copy_balance(dtq_qlinear_s* h, const dtq_balance* bal, cudaStream_t st) {
  if (!bal) return DTQ_OK;
  const int64_t K = h->K;
  if (bal->smooth) {
    CUDA_TRY(cudaMalloc(&h->smooth, K * sizeof(double)));
    CUDA_TRY(cudaMemcpyAsync(h->smooth, bal->smooth, K * sizeof(double),
                             cudaMemcpyDeviceToDevice, st));
  }
  if (bal->signs) {
    if (bal->hblock < 8 || bal->hblock > kMaxHblock || (bal->hblock & (bal->hblock - 1)) != 0)
      return fail(DTQ_ERR_INVALID_ARGUMENT, "hadamard: block must be a power of two in [8, %d]",
                  kMaxHblock);
    if (K % bal->hblock != 0)
      return fail(DTQ_ERR_INVALID_ARGUMENT, "rotate_channels: K not a multiple of the block");
    CUDA_TRY(cudaMalloc(&h->signs, K));
    CUDA_TRY(cudaMemcpyAsync(h->signs, bal->signs, K, cudaMemcpyDeviceToDevice, st));
    h->hblock = bal->hblock;
  }
  if ((h->smooth || h->signs) && h->hblock <= kMaxFusedHblock) {
    CUDA_TRY(cudaMalloc(&h->col_mul, K * sizeof(float)));
    col_mul_kernel<<<static_cast<int>((K + 255) / 256), 256, 0, st>>>(h->smooth, h->signs,
                                                                       h->hblock, K, h->col_mul);
    CUDA_TRY(cudaGetLastError());
  }
  return DTQ_OK;
}

int overflow_check(int abits, int wbits, int64_t K) {
  // int32 accumulation must be exact: (2^ab - 1) * 2^(wb-1) * K < 2^31.
  // W4 weights enter the MMA as 16*w (qgemm_sm100.cuh), i.e. with the W8 bound.
  if (wbits == 4) wbits = 8;
  const int64_t max_term = static_cast<int64_t>((1 << abits) - 1) * (int64_t{1} << (wbits - 1));
  if (max_term * K > INT32_MAX)
    return fail(DTQ_ERR_OVERFLOW, "qlinear_forward: accumulator could overflow (K=%lld)",
                (long long)K);
  return DTQ_OK;
}

// codes [N, ldc] (reference convention) + scale [N] -> handle weights
int finish_from_codes(dtq_qlinear_s* h, const uint8_t* codes, int64_t ldc, const double* scale,
                      const double* bias, cudaStream_t st) {
  const int64_t N = h->N, K = h->K;
  if (h->wbits != 4) {
    h->ld8 = round_up(K, 16);
    CUDA_TRY(cudaMalloc(&h->w8, N * h->ld8));
  } else {
    h->ld4 = round_up((K + 1) / 2, 16);
    CUDA_TRY(cudaMalloc(&h->w4, N * h->ld4));
  }
  CUDA_TRY(cudaMalloc(&h->wsum, N * sizeof(int32_t)));
  weight_pack_kernel<<<static_cast<int>(N), 256, 0, st>>>(codes, ldc, N, K, h->wbits, h->w8,
                                                          h->ld8, h->w4, h->ld4, h->wsum);
  CUDA_TRY(cudaGetLastError());
  if (scale != h->s_w) {
    CUDA_TRY(cudaMalloc(&h->s_w, N * sizeof(double)));
    CUDA_TRY(cudaMemcpyAsync(h->s_w, scale, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  CUDA_TRY(cudaMalloc(&h->s_w_f, N * sizeof(float)));
  const int g = static_cast<int>((N + 255) / 256);
  to_f32_kernel<<<g, 256, 0, st>>>(h->s_w, h->s_w_f, N, 0);
  CUDA_TRY(cudaGetLastError());
  if (bias) {
    CUDA_TRY(cudaMalloc(&h->bias, N * sizeof(double)));
    CUDA_TRY(cudaMalloc(&h->bias_f, N * sizeof(float)));
    CUDA_TRY(cudaMemcpyAsync(h->bias, bias, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
    to_f32_kernel<<<g, 256, 0, st>>>(h->bias, h->bias_f, N, 0);
    CUDA_TRY(cudaGetLastError());
  }
  const int rows[3] = {256, 128, 64};
  for (int i = 0; i < 3; ++i) {
    if (h->wbits != 4)
      DTQ_TRY(make_tmap_u8(&h->tmB[i], h->w8, N, K, h->ld8, dtq_gemm::BK, rows[i],
                           CU_TENSOR_MAP_SWIZZLE_128B));
    else
      // the nibble layout fills whole 8-column words (padding codes are 8 ->
      // zero), so the row's bytes run to 4 * ceil(K / 8), past (K + 1) / 2
      DTQ_TRY(make_tmap_u8(&h->tmB[i], h->w4, N, round_up(K, 8) / 2, h->ld4, dtq_gemm::BK / 2,
                           rows[i], CU_TENSOR_MAP_SWIZZLE_NONE));
  }
  return DTQ_OK;
}

// ------------------------------------------------------------------ GEMM launch
// (kernel instantiations live in gemm_w8.cu / gemm_w4.cu)
// Tile configuration: minimise (waves x per-SM tile width) over the candidate
// shapes; ties go to the CTA pair (half the B traffic per SM) and wider N.
// DTQ_GEMM_CFG=<0..3> forces {1cta/256, 1cta/128, 2cta/256, 2cta/128}.
GemmCfg choose_gemm_cfg(int64_t M, int64_t N, int wbits, int sms) {
  // preference order on ties: CTA pairs, then wide tiles
  const GemmCfg cands[4] = {{256, 1}, {256, 0}, {128, 1}, {128, 0}};
  static const int forced = [] {
    const char* e = std::getenv("DTQ_GEMM_CFG");
    return e ? std::atoi(e) : -1;
  }();
  if (forced >= 0 && forced < 4) {
    const GemmCfg f[4] = {{256, 0}, {128, 0}, {256, 1}, {128, 1}};
    return f[forced];
  }
  // W4A8 stays on single-CTA tiles (bound by the nibble unpack; pairs
  // measure slower: 1389 vs 1820 TOPS at C3 fc1), DTQ_GEMM_W4_CTA2=1
  // (diagnostics) lets the cost model below pick pairs for it.  Of the
  // single-CTA shapes, the two-M-sub-tile BN=128 one wins for N <= 2304
  // (proj 1606 vs 1460, fc2 2069 vs 1770 TOPS) and BN=256 for wide N
  // (fc1 1790 vs 1661 at C3).
  static const bool w4_cta2 = [] {
    const char* e = std::getenv("DTQ_GEMM_W4_CTA2");
    return e && e[0] == '1';
  }();
  if (wbits == 4 && !w4_cta2 && dtq_gemm::dual_m<128, true, false>()) {
    // both shapes do 256 x 128 x K (two sub-tiles) or 128 x 256 x K per tile:
    // fewer waves wins, then the N rule
    const int64_t w_dual = ((M + 255) / 256 * ((N + 127) / 128) + sms - 1) / sms;
    const int64_t w_256 = ((M + 127) / 128 * ((N + 255) / 256) + sms - 1) / sms;
    if (w_dual != w_256) return w_dual < w_256 ? GemmCfg{128, 0} : GemmCfg{256, 0};
    return N <= 2304 ? GemmCfg{128, 0} : GemmCfg{256, 0};
  }
  GemmCfg best{256, 0};
  int64_t best_cost = INT64_MAX;
  for (const GemmCfg& c : cands) {
    if (wbits == 4 && c.cta2 && !w4_cta2) continue;
    const bool m2 = wbits == 4 && !c.cta2 && c.bn == 128 && dtq_gemm::dual_m<128, true, false>();
    const int64_t tm = (c.cta2 || m2) ? 256 : 128;
    const int64_t tiles = ((M + tm - 1) / tm) * ((N + c.bn - 1) / c.bn);
    const int64_t units = c.cta2 ? sms / 2 : sms;
    const int64_t waves = (tiles + units - 1) / units;
    // a tile costs its BN columns plus a fixed ~128-column share (A-tile
    // loads, TMEM drain, epilogue tail): measured on the STDiT shapes, BN=256
    // CTA pairs win whenever the wave counts are within that margin
    const int64_t cost = waves * (c.bn + 128);
    if (cost < best_cost) {
      best_cost = cost;
      best = c;
    }
  }
  return best;
}

// diagnostics: device buffer of per-CTA wait-cycle counters, allocated only
// when DTQ_DEBUG_GEMM_PROBE=1 (read back with dtq_diag_probe_ptr)
unsigned long long* probe_buffer() {
  static unsigned long long* p = [] {
    const char* e = std::getenv("DTQ_DEBUG_GEMM_PROBE");
    unsigned long long* b = nullptr;
    if (e && e[0] == '1' && cudaMalloc(&b, 4096 * 8 * 8) == cudaSuccess)
      cudaMemset(b, 0, 4096 * 8 * 8);
    return b;
  }();
  return p;
}

int qgemm_impl(const uint8_t* codes, int64_t ldc, const double* s_x, const int32_t* z_x,
               int64_t M, dtq_qlinear_s* h, void* y, int y_dtype, int64_t ldy, cudaStream_t st,
               uint32_t* ready = nullptr, int act = DTQ_ACT_NONE,
               const int8_t* w8_tmp = nullptr) {
  if (act != DTQ_ACT_NONE && act != DTQ_ACT_GELU)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: bad activation %d", act);
  if (act != DTQ_ACT_NONE && !(y_dtype == DTQ_F16 || y_dtype == DTQ_BF16))
    return fail(DTQ_ERR_UNSUPPORTED, "qgemm: the activation epilogue writes F16 / BF16 only");
  if (!h) return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: null handle");
  if (M <= 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: M must be >= 1");
  if (!codes || !s_x || !z_x || !y) return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: null pointer");
  if (ldy < h->N) return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: ldy < N");
  if (M > INT32_MAX / 2) return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: M too large");
  DTQ_TRY(overflow_check(h->abits, h->wbits, h->K));
  DTQ_TRY(check_device());
  const int sms = device_info().sms;
  // w8_tmp: W4A8 weights unpacked to s8 by this forward (w4_unpack_kernel):
  // the W8A8 kernels run on them, B read after griddepcontrol.wait
  const int wbits = w8_tmp ? 8 : h->wbits;
  const GemmCfg cfg = choose_gemm_cfg(M, h->N, wbits, sms);
  const int BN = cfg.bn;
  const bool m2 = wbits == 4 && !cfg.cta2 && cfg.bn == 128 &&
                  dtq_gemm::dual_m<128, true, false>();  // two M sub-tiles per CTA
  const int tile_m = (cfg.cta2 || m2) ? 2 * dtq_gemm::BM : dtq_gemm::BM;
  const int brows = cfg.cta2 ? BN / 2 : BN;
  CUtensorMap tB = h->tmB[brows == 256 ? 0 : (brows == 128 ? 1 : 2)];
  if (w8_tmp)
    DTQ_TRY(cached_tmap_u8(h, &tB, w8_tmp, h->N, h->K, round_up(h->K, 16), dtq_gemm::BK, brows,
                           CU_TENSOR_MAP_SWIZZLE_128B));

  CUtensorMap tA;
  DTQ_TRY(cached_tmap_u8(h, &tA, codes, M, h->K, ldc, dtq_gemm::BK, dtq_gemm::BM,
                         CU_TENSOR_MAP_SWIZZLE_128B));

  void* yk = y;
  int64_t ldk = ldy;
  int kind;
  switch (y_dtype) {
    case DTQ_F16: kind = dtq_gemm::kOutF16; break;
    case DTQ_BF16: kind = dtq_gemm::kOutBF16; break;
    case DTQ_F32: kind = dtq_gemm::kOutF32; break;
    case DTQ_S32: kind = dtq_gemm::kOutS32; break;
    case DTQ_F64:
      kind = dtq_gemm::kOutS32;
      DTQ_TRY(grow(reinterpret_cast<void**>(&h->acc32), &h->acc32_bytes,
                   static_cast<size_t>(M) * h->N * sizeof(int32_t)));
      yk = h->acc32;
      ldk = h->N;
      break;
    default: return fail(DTQ_ERR_INVALID_ARGUMENT, "qgemm: bad output dtype %d", y_dtype);
  }
  const size_t es = kind == dtq_gemm::kOutF16 || kind == dtq_gemm::kOutBF16 ? 2 : 4;

  dtq_gemm::GemmArgs g{};
  g.M = static_cast<int>(M);
  g.N = static_cast<int>(h->N);
  g.K = static_cast<int>(h->K);
  g.tiles_m = static_cast<int>((M + tile_m - 1) / tile_m);
  g.tiles_n = static_cast<int>((h->N + BN - 1) / BN);
  g.k_blocks = static_cast<int>((h->K + dtq_gemm::BK - 1) / dtq_gemm::BK);
  g.s_x = s_x;
  g.z_x = z_x;
  g.s_w = h->s_w_f;
  g.wsum = h->wsum;
  g.bias = kind == dtq_gemm::kOutS32 ? nullptr : h->bias_f;
  g.y = yk;
  g.ldy = ldk;
  // diagnostics: DTQ_DEBUG_GEMM_NOEPI=1 runs the main loop without an epilogue
  static const bool noepi = [] {
    const char* e = std::getenv("DTQ_DEBUG_GEMM_NOEPI");
    return e && e[0] == '1';
  }();
  g.out_kind = noepi ? dtq_gemm::kOutNone : kind;
  static const int dbg = [] {
    const char* e = std::getenv("DTQ_DEBUG_GEMM_EPI");
    return e ? std::atoi(e) : 0;
  }();
  g.dbg = dbg;
  g.probe = probe_buffer();
  g.w4 = h->w4;
  g.ld4 = h->ld4;
  // row flags (forward_impl, when the tile quantizer runs beside this GEMM)
  g.ready = ready;
  g.done = ready ? ready + kMaxFlagBlocks : nullptr;
  g.mblocks = static_cast<int>((M + 127) / 128);
  g.act = act;
  g.b_pre = w8_tmp ? 0 : 1;
  static const bool no_tma_store = [] {
    const char* e = std::getenv("DTQ_DEBUG_NO_TMA_STORE");
    return e && e[0] == '1';
  }();
  g.tma_store = !no_tma_store && (reinterpret_cast<uintptr_t>(yk) % 16 == 0) &&
                ((ldk * es) % 16 == 0);
  CUtensorMap tY;
  std::memset(&tY, 0, sizeof(tY));
  if (g.tma_store)
    DTQ_TRY(cached_tmap_u8(h, &tY, yk, M, h->N * static_cast<int64_t>(es), ldk * es, 64, 32,
                           CU_TENSOR_MAP_SWIZZLE_64B));

  const cudaError_t e = ready ? dtq_launch_gemm_w8_cores(tA, tB, tY, g, cfg, sms, st)
                       : wbits != 4 ? dtq_launch_gemm_w8(tA, tB, tY, g, cfg, sms, st)
                                       : dtq_launch_gemm_w4(tA, tB, tY, g, cfg, sms, st);
  if (e != cudaSuccess) return fail(DTQ_ERR_CUDA, "qgemm launch: %s", cudaGetErrorString(e));

  if (y_dtype == DTQ_F64) {
    const int64_t total = M * h->N;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    parity_epilogue_kernel<<<grid, 256, 0, st>>>(
        h->acc32, M, h->N, s_x, h->s_w, h->bias, static_cast<double*>(y), ldy);
    CUDA_TRY(cudaGetLastError());
  }
  return DTQ_OK;
}

// workspace: [row-flag counters: kMaxFlagBlocks + the GEMM's exit ticket]
// [codes M x ldc][s_x f64 M][z_x i32 M] and, for W4A8 handles, [s8 weights
// N x round_up(K, 16)] (w4_unpack_kernel).  The counter region has a fixed
// size (a workspace serves forwards of any M) and must be zero before first
// use; every forward leaves it zero.
constexpr size_t kFlagBytes = (kMaxFlagBlocks + 64) * sizeof(uint32_t);
size_t ws_layout(const dtq_qlinear_s* h, int64_t M, int64_t* ldc, size_t* off_codes,
                 size_t* off_s, size_t* off_z, size_t* off_w = nullptr) {
  *ldc = round_up(h->K, 16);
  *off_codes = kFlagBytes;
  const size_t codes = kFlagBytes + round_up(static_cast<int64_t>(M) * *ldc, 256);
  *off_s = codes;
  *off_z = codes + round_up(M * 8, 256);
  const size_t end = *off_z + round_up(M * 4, 256);
  if (off_w) *off_w = h->wbits == 4 ? end : 0;
  return end + (h->wbits == 4 ? round_up(h->N * round_up(h->K, 16), 256) : 0);
}

// W4A8 forward through s8 weights unpacked into the workspace (then the
// W8A8 kernels, CTA pairs included) rather than the GEMM's in-kernel
// unpack.  DTQ_W4_UNPACK=0 / 1 (diagnostics) forces either.
bool w4_unpack_wanted(const dtq_qlinear_s* h, int64_t M) {
  static const int forced = [] {
    const char* e = std::getenv("DTQ_W4_UNPACK");
    return e ? std::atoi(e) : -1;
  }();
  if (h->wbits != 4) return false;
  if (forced >= 0) return forced != 0;
  (void)M;
  return true;
}

dtq_w4::Unpack w4_job(const dtq_qlinear_s* h, int8_t* out) {
  dtq_w4::Unpack u;
  u.src = h->w4;
  u.ld4 = h->ld4;
  u.rows = h->N;
  u.chunks = (round_up(h->K, 8) / 2 + 15) / 16;
  u.dst = out;
  u.ld8 = round_up(h->K, 16);
  return u;
}

int launch_w4_unpack(const dtq_w4::Unpack& u, cudaStream_t st) {
  const int64_t total = u.rows * u.chunks;
  const int64_t cap = static_cast<int64_t>(device_info().sms) * 8;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, cap)));
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, w4_unpack_kernel, u);
  if (e != cudaSuccess) return fail(DTQ_ERR_CUDA, "w4 unpack launch: %s", cudaGetErrorString(e));
  return DTQ_OK;
}

// Row flags for this forward?  The quantizer and the GEMM then run
// concurrently, one CTA of each per SM (W8A8 with an fp32 epilogue output;
// the tile quantizer; both fitting an SM -- checked by the launcher).
// Opt-in (DTQ_ROW_FLAGS=1): measured SLOWER than the two stages back to back
// on the C2 step (35.3 vs 28.3 us per forward in a CUDA graph,
// profiles/r02_rowflags.md).  Programmatic launch does co-schedule the GEMM
// beside the quantizer, but each forward's quantizer still waits for the
// whole previous GEMM (its input may be that GEMM's output), the GEMM's CTAs
// need the SM space the previous GEMM's tail CTAs hold, and the quantizer at
// one CTA per SM is ~1.4x slower -- the overlap it buys is smaller than what
// it costs.  Kept, tested (tests/test_gpu_rowflags.py), off by default.
bool row_flags_wanted(const dtq_qlinear_s* h, int64_t M, int y_dtype) {
  static const bool on = [] {
    const char* e = std::getenv("DTQ_ROW_FLAGS");
    return e != nullptr && e[0] == '1';
  }();
  return on && h->wbits != 4 && (M + 127) / 128 <= kMaxFlagBlocks &&
         (y_dtype == DTQ_F16 || y_dtype == DTQ_BF16 || y_dtype == DTQ_F32);
}

int forward_impl(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_s* h, int mode,
                 const dtq_prologue* pro, void* y, int y_dtype, int64_t ldy, void* ws,
                 size_t ws_bytes, int32_t* status, cudaStream_t st, int act = DTQ_ACT_NONE) {
  if (!h) return fail(DTQ_ERR_INVALID_ARGUMENT, "forward: null handle");
  if (ldx < h->K) return fail(DTQ_ERR_INVALID_ARGUMENT, "qlinear_forward: X cols != C_in");
  int64_t ldc;
  size_t off_c, off_s, off_z, off_w;
  const size_t need = ws_layout(h, M, &ldc, &off_c, &off_s, &off_z, &off_w);
  if (!ws) {
    DTQ_TRY(grow(&h->scratch, &h->scratch_bytes, need, st, true));
    ws = h->scratch;
  } else if (ws_bytes < need) {
    return fail(DTQ_ERR_INVALID_ARGUMENT, "forward: workspace too small (%zu < %zu)", ws_bytes,
                need);
  } else if (reinterpret_cast<uintptr_t>(ws) % 16 != 0) {
    // the codes and the W4A8 s8 weights are TMA operands
    return fail(DTQ_ERR_INVALID_ARGUMENT, "forward: workspace must be 16-byte aligned");
  }
  uint8_t* base = static_cast<uint8_t*>(ws);
  uint32_t* ready = reinterpret_cast<uint32_t*>(base);
  uint8_t* codes = base + off_c;
  double* s_x = reinterpret_cast<double*>(base + off_s);
  int32_t* z_x = reinterpret_cast<int32_t*>(base + off_z);
  DTQ_TRY(overflow_check(h->abits, h->wbits, h->K));
  // W4A8: s8 weights expanded into the workspace by the quantizer's CTAs, or
  // by their own kernel between the quantizer and the GEMM
  int8_t* w8_tmp = w4_unpack_wanted(h, M) ? reinterpret_cast<int8_t*>(base + off_w) : nullptr;
  const dtq_w4::Unpack w4u = w8_tmp ? w4_job(h, w8_tmp) : dtq_w4::Unpack{};
  int w4_done = 0;
  int p_regs = 0, p_smem = 0, flags = 0;
  if (act == DTQ_ACT_NONE && row_flags_wanted(h, M, y_dtype)) {
    DTQ_TRY(check_device());
    const GemmCfg cfg = choose_gemm_cfg(M, h->N, h->wbits, device_info().sms);
    const int kind = y_dtype == DTQ_F16 ? dtq_gemm::kOutF16
                     : y_dtype == DTQ_BF16 ? dtq_gemm::kOutBF16 : dtq_gemm::kOutF32;
    if (dtq_gemm_w8_cores_info(cfg, kind, &p_regs, &p_smem) != 0) ready = nullptr;
  } else {
    ready = nullptr;
  }
  DTQ_TRY(quantize_rows_impl(x, x_dtype, M, h->K, ldx, h->abits, 0, mode, 0, h->smooth,
                             h->col_mul, h->signs, h->hblock, pro, codes, ldc, s_x, z_x,
                             status, st, true, ready, p_regs, p_smem, &flags,
                             w8_tmp ? &w4u : nullptr, &w4_done));
  if (w8_tmp && !w4_done) DTQ_TRY(launch_w4_unpack(w4u, st));
  return qgemm_impl(codes, ldc, s_x, z_x, M, h, y, y_dtype, ldy, st, flags ? ready : nullptr, act,
                    w8_tmp);
}

}  // namespace

// one MixedPrecisionPlan row on the device: a handle per distinct bit width
constexpr int kPlanRanges = 4;  // plan.hpp:17 kNumRanges
struct dtq_planned_s {
  int bits[kPlanRanges] = {8, 8, 8, 8};
  dtq_qlinear_t range_handle[kPlanRanges] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<dtq_qlinear_t> owned;
};

namespace {

// ------------------------------------------------------------------ checkpoints
// Parser of the reference's quantized-checkpoint format (trace_io.cpp:
// 225-316), restated: little-endian fields read with bounds checks, every
// malformed input a DTQ_ERR_INVALID_ARGUMENT (the reference's FormatError).
struct CkptLayer {
  std::string name;
  int64_t N = 0, K = 0;
  int bits = 8;
  int grouping = 0;
  int64_t group_size = 0;
  bool symmetric = true;
  std::vector<float> scale;
  std::vector<int32_t> zero;
  std::vector<uint8_t> packed;  // LSB-first codes of all N*K weights
  std::vector<float> mask;
  std::vector<int8_t> rot;
};

struct CkptReader {
  const std::vector<char>& buf;
  size_t pos = 0;
  bool ok = true;
  template <typename T>
  T get() {
    T v{};
    if (pos + sizeof(T) > buf.size()) {
      ok = false;
      return v;
    }
    std::memcpy(&v, buf.data() + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  bool bytes(void* dst, size_t n) {
    if (pos + n > buf.size() || pos + n < pos) return ok = false;
    if (n) std::memcpy(dst, buf.data() + pos, n);
    pos += n;
    return true;
  }
};

}  // namespace

struct dtq_checkpoint_s {
  std::vector<CkptLayer> layers;
};

namespace {

int parse_checkpoint(const std::vector<char>& buf, dtq_checkpoint_s* ck) {
  static const char kMagic[8] = {'D', 'T', 'Q', 'C', 'K', 'P', 'T', '\0'};
  CkptReader r{buf};
  char magic[8];
  if (!r.bytes(magic, 8) || std::memcmp(magic, kMagic, 8) != 0)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint magic mismatch");
  const uint16_t version = r.get<uint16_t>();
  if (!r.ok || version != 1)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "unsupported checkpoint format version %u", version);
  const uint32_t n = r.get<uint32_t>();
  if (!r.ok) return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated checkpoint header");
  for (uint32_t i = 0; i < n; ++i) {
    CkptLayer L;
    const uint16_t name_len = r.get<uint16_t>();
    L.name.resize(name_len);
    if (!r.ok || !r.bytes(L.name.data(), name_len))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer name (layer %u)", i);
    L.N = r.get<uint32_t>();
    L.K = r.get<uint32_t>();
    L.bits = r.get<uint8_t>();
    L.grouping = r.get<uint8_t>();
    L.group_size = r.get<uint32_t>();
    L.symmetric = r.get<uint8_t>() != 0;
    const uint32_t n_params = r.get<uint32_t>();
    if (!r.ok) return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer header (layer %u)", i);
    if (!bits_supported(L.bits))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint with unsupported bits (%d)", L.bits);
    L.scale.resize(n_params);
    if (!r.bytes(L.scale.data(), 4ull * n_params))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer params (layer %u)", i);
    if (!L.symmetric) {
      L.zero.resize(n_params);
      if (!r.bytes(L.zero.data(), 4ull * n_params))
        return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer params (layer %u)", i);
    }
    const uint64_t packed_len = r.get<uint64_t>();
    const uint64_t want = (static_cast<uint64_t>(L.N) * L.K * L.bits + 7) / 8;
    if (!r.ok || packed_len != want)
      return fail(DTQ_ERR_INVALID_ARGUMENT, "bad packing length (layer %u)", i);
    L.packed.resize(packed_len);
    if (!r.bytes(L.packed.data(), packed_len))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer weights (layer %u)", i);
    const uint32_t mask_len = r.get<uint32_t>();
    L.mask.resize(r.ok ? mask_len : 0);
    if (!r.ok || !r.bytes(L.mask.data(), 4ull * mask_len))
      return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer mask (layer %u)", i);
    const uint32_t rot_len = r.get<uint32_t>();
    if (!r.ok) return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer rotation (layer %u)", i);
    if (rot_len > 0) {
      std::vector<uint8_t> bitsv((rot_len + 7) / 8);
      if (!r.bytes(bitsv.data(), bitsv.size()))
        return fail(DTQ_ERR_INVALID_ARGUMENT, "truncated layer rotation (layer %u)", i);
      L.rot.resize(rot_len);
      for (uint32_t j = 0; j < rot_len; ++j) L.rot[j] = ((bitsv[j / 8] >> (j % 8)) & 1) ? 1 : -1;
    }
    ck->layers.push_back(std::move(L));
  }
  if (r.pos != buf.size()) return fail(DTQ_ERR_INVALID_ARGUMENT, "trailing bytes after last layer");
  return DTQ_OK;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* dtq_last_error(void) { return g_last_error.c_str(); }

int dtq_capi_version(void) { return DTQ_CAPI_VERSION; }

int dtq_device_check(void) { return check_device(); }

// diagnostics only (deliberately not declared in include/dtq_capi.h)
void* dtq_diag_probe_ptr(void) { return probe_buffer(); }
void* dtq_diag_fq_probe_ptr(void) { return fq_probe_buffer(); }

int dtq_quantize_rows(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                      int bits, int symmetric, int mode, const dtq_balance* balance,
                      const dtq_prologue* prologue, uint8_t* codes, int64_t ldc, double* scale,
                      int32_t* zero, int32_t* status, void* stream) {
  NvtxRange nvtx_range("dtq_quantize_rows");
  const double* smooth = balance ? balance->smooth : nullptr;
  const int8_t* signs = balance ? balance->signs : nullptr;
  const int hblock = balance ? balance->hblock : 0;
  cudaStream_t st = as_stream(stream);
  float* mulv = nullptr;
  if (signs && hblock > kMaxFusedHblock) mode = DTQ_MODE_EXACT;  // the fp64 pre-pass
  const bool exact = mode == DTQ_MODE_EXACT || x_dtype == DTQ_F64;
  if ((smooth || signs) && !exact) {
    // fast mode folds sign / smooth / norm into one fp32 multiplier: derive it
    // stream-ordered for this call
    if (cols <= 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: empty matrix");
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&mulv), cols * sizeof(float), st));
    col_mul_kernel<<<static_cast<int>((cols + 255) / 256), 256, 0, st>>>(smooth, signs, hblock,
                                                                          cols, mulv);
    CUDA_TRY(cudaGetLastError());
  }
  const int r = quantize_rows_impl(x, x_dtype, rows, cols, ldx, bits, symmetric, mode, 0,
                                   exact ? smooth : nullptr, mulv, signs, hblock, prologue,
                                   codes, ldc, scale, zero, status, st,
                                   /*col_mul_const=*/mulv == nullptr);
  if (mulv) cudaFreeAsync(mulv, st);
  return r;
}

int dtq_qlinear_create(const void* w, int w_dtype, int64_t N, int64_t K, int64_t ldw,
                       int weight_bits, int act_bits, const double* bias,
                       const dtq_balance* balance, void* stream, dtq_qlinear_t* out) {
  NvtxRange nvtx_range("dtq_qlinear_create");
  if (!out) return fail(DTQ_ERR_INVALID_ARGUMENT, "create: null out");
  *out = nullptr;
  if (!bits_supported(weight_bits))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "make_quant_linear: unsupported bit width");
  if (!bits_supported(act_bits))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "make_quant_linear: unsupported bit width");
  if (N <= 0 || K <= 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "make_quant_linear: empty W");
  DTQ_TRY(check_device());
  cudaStream_t st = as_stream(stream);
  auto* h = new dtq_qlinear_s();
  h->N = N;
  h->K = K;
  h->wbits = weight_bits;
  h->abits = act_bits;
  int r = alloc_status(h, st);
  if (r == DTQ_OK) r = copy_balance(h, balance, st);
  uint8_t* codes = nullptr;
  if (r == DTQ_OK) {
    const int64_t ldc = round_up(K, 16);
    if (cudaMalloc(&codes, N * ldc) != cudaSuccess ||
        cudaMalloc(&h->s_w, N * sizeof(double)) != cudaSuccess) {
      r = fail(DTQ_ERR_CUDA, "create: out of device memory");
    } else {
      int32_t* zw = nullptr;
      if (cudaMalloc(&zw, N * sizeof(int32_t)) != cudaSuccess) {
        r = fail(DTQ_ERR_CUDA, "create: out of device memory");
      } else {
        // weight side of apply_balance: W * s then the rotation, in fp64; then
        // symmetric per-output-channel quantization (make_quant_linear)
        r = quantize_rows_impl(w, w_dtype, N, K, ldw, weight_bits, 1, DTQ_MODE_EXACT, 1,
                               h->smooth, nullptr, h->signs, h->hblock, nullptr, codes, ldc,
                               h->s_w, zw, h->status, st);
        if (r == DTQ_OK) {
          int32_t bad = 0;
          if (cudaMemcpyAsync(&bad, h->status, sizeof(int32_t), cudaMemcpyDeviceToHost, st) !=
                  cudaSuccess ||
              cudaStreamSynchronize(st) != cudaSuccess)
            r = fail(DTQ_ERR_CUDA, "create: status readback failed");
          else if (bad)
            r = fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: non-finite value in group");
        }
        cudaFreeAsync(zw, st);
      }
      if (r == DTQ_OK) r = finish_from_codes(h, codes, ldc, h->s_w, bias, st);
    }
  }
  if (codes) cudaFreeAsync(codes, st);
  if (r != DTQ_OK) {
    free_handle(h);
    return r;
  }
  *out = h;
  return DTQ_OK;
}

int dtq_qlinear_create_from_codes(const uint8_t* codes, int packed, int64_t ld, int weight_bits,
                                  const double* scale, int64_t N, int64_t K, int act_bits,
                                  const double* bias, const dtq_balance* balance, void* stream,
                                  dtq_qlinear_t* out) {
  NvtxRange nvtx_range("dtq_qlinear_create_from_codes");
  if (!out) return fail(DTQ_ERR_INVALID_ARGUMENT, "create: null out");
  *out = nullptr;
  if (!bits_supported(weight_bits))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "unsupported bit width");
  if (!bits_supported(act_bits)) return fail(DTQ_ERR_INVALID_ARGUMENT, "unsupported bit width");
  if (N <= 0 || K <= 0 || !codes || !scale)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "create_from_codes: bad arguments");
  if (!packed && ld < K) return fail(DTQ_ERR_INVALID_ARGUMENT, "create_from_codes: ld < K");
  DTQ_TRY(check_device());
  cudaStream_t st = as_stream(stream);
  auto* h = new dtq_qlinear_s();
  h->N = N;
  h->K = K;
  h->wbits = weight_bits;
  h->abits = act_bits;
  int r = alloc_status(h, st);
  if (r == DTQ_OK) r = copy_balance(h, balance, st);
  uint8_t* tmp = nullptr;
  const uint8_t* src = codes;
  int64_t lds = ld;
  if (r == DTQ_OK && packed) {
    lds = K;
    if (cudaMalloc(&tmp, N * K) != cudaSuccess) {
      r = fail(DTQ_ERR_CUDA, "create_from_codes: out of device memory");
    } else {
      const int64_t count = N * K;
      const int grid = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 32));
      unpack_stream_kernel<<<grid, 256, 0, st>>>(codes, count, weight_bits, N, K, tmp, K);
      if (cudaGetLastError() != cudaSuccess) r = fail(DTQ_ERR_CUDA, "unpack launch failed");
      src = tmp;
    }
  }
  if (r == DTQ_OK) r = finish_from_codes(h, src, lds, scale, bias, st);
  if (tmp) cudaFreeAsync(tmp, st);
  if (r != DTQ_OK) {
    free_handle(h);
    return r;
  }
  *out = h;
  return DTQ_OK;
}

int dtq_qlinear_destroy(dtq_qlinear_t h) {
  if (h) free_handle(h);
  return DTQ_OK;
}

int dtq_qlinear_info(dtq_qlinear_t h, int64_t* N, int64_t* K, int* wbits, int* abits) {
  if (!h) return fail(DTQ_ERR_INVALID_ARGUMENT, "info: null handle");
  if (N) *N = h->N;
  if (K) *K = h->K;
  if (wbits) *wbits = h->wbits;
  if (abits) *abits = h->abits;
  return DTQ_OK;
}

int dtq_qlinear_export(dtq_qlinear_t h, uint8_t* codes, double* scale, int32_t* wsum,
                       void* stream) {
  if (!h) return fail(DTQ_ERR_INVALID_ARGUMENT, "export: null handle");
  cudaStream_t st = as_stream(stream);
  if (codes) {
    uint8_t* tmp = nullptr;
    CUDA_TRY(cudaMalloc(&tmp, h->N * h->K));
    const int grid = static_cast<int>(std::min<int64_t>((h->N * h->K + 255) / 256, 148 * 32));
    export_codes_kernel<<<grid, 256, 0, st>>>(h->w8, h->ld8, h->w4, h->ld4, h->wbits, h->N, h->K,
                                              tmp);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(codes, tmp, h->N * h->K, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(tmp);
  }
  if (scale) CUDA_TRY(cudaMemcpyAsync(scale, h->s_w, h->N * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (wsum) CUDA_TRY(cudaMemcpyAsync(wsum, h->wsum, h->N * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DTQ_OK;
}

int dtq_qgemm(const uint8_t* codes, int64_t ldc, const double* s_x, const int32_t* z_x, int64_t M,
              dtq_qlinear_t h, void* y, int y_dtype, int64_t ldy, void* stream) {
  NvtxRange nvtx_range("dtq_qgemm");
  return qgemm_impl(codes, ldc, s_x, z_x, M, h, y, y_dtype, ldy, as_stream(stream));
}

size_t dtq_qlinear_workspace_bytes(dtq_qlinear_t h, int64_t M) {
  if (!h || M <= 0) return 0;
  int64_t ldc;
  size_t a, b, c;
  return ws_layout(h, M, &ldc, &a, &b, &c);
}

int dtq_qlinear_forward(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                        int mode, const dtq_prologue* prologue, void* y, int y_dtype,
                        int64_t ldy, void* workspace, size_t workspace_bytes, int32_t* status,
                        void* stream) {
  NvtxRange nvtx_range("dtq_qlinear_forward");
  return forward_impl(x, x_dtype, M, ldx, h, mode, prologue, y, y_dtype, ldy, workspace,
                      workspace_bytes, status, as_stream(stream));
}

int dtq_qlinear_forward_act(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                            int mode, const dtq_prologue* prologue, int activation, void* y,
                            int y_dtype, int64_t ldy, void* workspace, size_t workspace_bytes,
                            int32_t* status, void* stream) {
  NvtxRange nvtx_range("dtq_qlinear_forward_act");
  if (activation != DTQ_ACT_NONE && activation != DTQ_ACT_GELU)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "forward: bad activation %d", activation);
  return forward_impl(x, x_dtype, M, ldx, h, mode, prologue, y, y_dtype, ldy, workspace,
                      workspace_bytes, status, as_stream(stream), activation);
}

int dtq_qlinear_quantize(const void* x, int x_dtype, int64_t M, int64_t ldx, dtq_qlinear_t h,
                         int mode, const dtq_prologue* prologue, uint8_t* codes, int64_t ldc,
                         double* scale, int32_t* zero, int32_t* status, void* stream) {
  NvtxRange nvtx_range("dtq_qlinear_quantize");
  if (!h) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: null handle");
  if (ldx < h->K) return fail(DTQ_ERR_INVALID_ARGUMENT, "qlinear_forward: X cols != C_in");
  return quantize_rows_impl(x, x_dtype, M, h->K, ldx, h->abits, 0, mode, 0, h->smooth,
                            h->col_mul, h->signs, h->hblock, prologue, codes, ldc, scale, zero,
                            status, as_stream(stream));
}

int dtq_qlinear_forward_host(const void* x, int x_dtype, int64_t M, dtq_qlinear_t h, int mode,
                             void* y, int y_dtype, void* stream) {
  NvtxRange nvtx_range("dtq_qlinear_forward_host");
  if (!h || !x || !y || M <= 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "forward_host: bad args");
  const size_t xe = dtype_size(x_dtype), ye = dtype_size(y_dtype);
  const size_t xb = xe * static_cast<size_t>(M) * h->K;
  const size_t yb = ye * static_cast<size_t>(M) * h->N;
  if (xb == 0 || yb == 0) return fail(DTQ_ERR_INVALID_ARGUMENT, "forward_host: bad dtype");
  cudaStream_t st = as_stream(stream);
  std::lock_guard<std::mutex> host_lock(h->host_mu);  // handle-owned buffers and streams
  DTQ_TRY(grow(&h->hx, &h->hx_bytes, xb));
  DTQ_TRY(grow(&h->hy, &h->hy_bytes, yb));
  CUDA_TRY(cudaMemsetAsync(h->status, 0, sizeof(int32_t), st));
  // Row chunks (multiples of 128 rows) in a three-stage pipeline: H2D on one
  // stream, quantize + GEMM of chunk i once its rows have landed, D2H of
  // chunk i once its GEMM is done, on a third stream (quantization is
  // row-local, so chunks are independent).  The D2H (the larger transfer:
  // N > K columns) should run back to back from as early as possible, so the
  // chunks grow geometrically: 128 rows first (its H2D and forward take
  // ~15 us), then doubling -- each chunk's H2D (K columns in, at the rate
  // left beside the D2H) lands before the D2H stream reaches it, with one H2D
  // and one D2H copy per chunk (few copies: every interleaved H2D copy costs
  // D2H rate).  DTQ_HOST_CHUNKS=n (diagnostics) uses n equal chunks instead.
  // The F64 parity output uses a handle-wide s32 scratch and stays in one
  // piece.
  static const int nchunks = [] {
    const char* e = std::getenv("DTQ_HOST_CHUNKS");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 0;
  }();
  std::vector<int64_t> rows_of;  // chunk sizes
  if (!(y_dtype == DTQ_F64 || M < 1024)) {
    if (nchunks > 0) {
      const int64_t c = ((M + nchunks - 1) / nchunks + 127) / 128 * 128;
      for (int64_t r = 0; r < M; r += c) rows_of.push_back(std::min(c, M - r));
    } else {
      // DTQ_HOST_FIRST / DTQ_HOST_GROWTH (diagnostics): first chunk, growth
      static const int64_t first = [] {
        const char* e = std::getenv("DTQ_HOST_FIRST");
        return e && std::atoll(e) >= 128 ? std::atoll(e) / 128 * 128 : 128;
      }();
      static const int64_t growth = [] {
        const char* e = std::getenv("DTQ_HOST_GROWTH");
        return e && std::atoll(e) >= 2 ? std::atoll(e) : 2;
      }();
      int64_t c = first;
      for (int64_t r = 0; r < M;) {
        int64_t m = std::min(c, M - r);
        if (M - r - m < c) m = M - r;  // a short remainder joins the last chunk
        rows_of.push_back(m);
        r += m;
        c *= growth;
      }
    }
  }
  if (rows_of.size() <= 1) {
    CUDA_TRY(cudaMemcpyAsync(h->hx, x, xb, cudaMemcpyHostToDevice, st));
    DTQ_TRY(forward_impl(h->hx, x_dtype, M, h->K, h, mode, nullptr, h->hy, y_dtype, h->N,
                         nullptr, 0, h->status, st));
    CUDA_TRY(cudaMemcpyAsync(y, h->hy, yb, cudaMemcpyDeviceToHost, st));
  } else {
    int64_t ldc;
    size_t a_, b_, c_;
    const int64_t max_rows = *std::max_element(rows_of.begin(), rows_of.end());
    const size_t wsb = ws_layout(h, max_rows, &ldc, &a_, &b_, &c_);
    DTQ_TRY(grow(&h->pws, &h->pws_bytes, wsb, st, true));
    for (cudaStream_t& s : h->ps)
      if (!s) CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    for (cudaEvent_t& e : h->pe)
      if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const size_t nc = rows_of.size();
    while (h->ev_in.size() < nc) {
      cudaEvent_t a, b;
      CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      h->ev_in.push_back(a);
      h->ev_out.push_back(b);
    }
    cudaStream_t s_in = h->ps[0], s_cmp = h->ps[1], s_out = h->ps[2];
    // DTQ_HOST_TRACE=1 (diagnostics): per-chunk stage completion times to stderr
    static const bool trace = [] {
      const char* e = std::getenv("DTQ_HOST_TRACE");
      return e && e[0] == '1';
    }();
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t s) {
      if (!trace) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, s);
      tev.push_back(e);
    };
    mark(st);
    CUDA_TRY(cudaEventRecord(h->pe[0], st));  // fork: after the status reset
    for (cudaStream_t s : h->ps) CUDA_TRY(cudaStreamWaitEvent(s, h->pe[0], 0));
    int64_t r0 = 0;
    for (size_t c = 0; c < nc; r0 += rows_of[c], ++c) {
      const int64_t m = rows_of[c];
      const size_t xo = xe * static_cast<size_t>(r0) * h->K, yo = ye * static_cast<size_t>(r0) * h->N;
      uint8_t* dx = static_cast<uint8_t*>(h->hx) + xo;
      uint8_t* dy = static_cast<uint8_t*>(h->hy) + yo;
      CUDA_TRY(cudaMemcpyAsync(dx, static_cast<const uint8_t*>(x) + xo, xe * m * h->K,
                               cudaMemcpyHostToDevice, s_in));
      CUDA_TRY(cudaEventRecord(h->ev_in[c], s_in));
      mark(s_in);
      CUDA_TRY(cudaStreamWaitEvent(s_cmp, h->ev_in[c], 0));
      DTQ_TRY(forward_impl(dx, x_dtype, m, h->K, h, mode, nullptr, dy, y_dtype, h->N, h->pws,
                           h->pws_bytes, h->status, s_cmp));
      CUDA_TRY(cudaEventRecord(h->ev_out[c], s_cmp));
      mark(s_cmp);
      CUDA_TRY(cudaStreamWaitEvent(s_out, h->ev_out[c], 0));
      CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t*>(y) + yo, dy, ye * m * h->N,
                               cudaMemcpyDeviceToHost, s_out));
      mark(s_out);
    }
    // join: the D2H stream finishes last (it waits on every GEMM, which waits
    // on every H2D)
    CUDA_TRY(cudaEventRecord(h->pe[1], s_out));
    CUDA_TRY(cudaStreamWaitEvent(st, h->pe[1], 0));
    if (trace) {
      cudaStreamSynchronize(st);
      std::string line = "forward_host trace (us from fork; in/gemm/out per chunk):";
      for (size_t k = 1; k < tev.size(); ++k) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[0], tev[k]);
        line += " " + std::to_string(static_cast<int>(ms * 1e3f));
      }
      fprintf(stderr, "%s\n", line.c_str());
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
  }
  int32_t bad = 0;
  CUDA_TRY(cudaMemcpyAsync(&bad, h->status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (bad) return fail(DTQ_ERR_INVALID_ARGUMENT, "quantize: non-finite input");
  return DTQ_OK;
}


int dtq_checkpoint_open(const char* path, dtq_checkpoint_t* out) {
  if (!out || !path) return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint_open: null argument");
  *out = nullptr;
  std::ifstream f(path, std::ios::binary);
  if (!f) return fail(DTQ_ERR_INVALID_ARGUMENT, "cannot open checkpoint %s", path);
  std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  auto* ck = new dtq_checkpoint_s();
  const int r = parse_checkpoint(buf, ck);
  if (r != DTQ_OK) {
    delete ck;
    return r;
  }
  *out = ck;
  return DTQ_OK;
}

int dtq_checkpoint_close(dtq_checkpoint_t ck) {
  delete ck;
  return DTQ_OK;
}

int dtq_checkpoint_num_layers(dtq_checkpoint_t ck, int64_t* n) {
  if (!ck || !n) return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint: null argument");
  *n = static_cast<int64_t>(ck->layers.size());
  return DTQ_OK;
}

int dtq_checkpoint_layer_info(dtq_checkpoint_t ck, int64_t i, const char** name, int64_t* N,
                              int64_t* K, int* bits, int* symmetric, int64_t* mask_len,
                              int64_t* rot_len) {
  if (!ck || i < 0 || i >= static_cast<int64_t>(ck->layers.size()))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint: bad layer index %lld", (long long)i);
  const CkptLayer& L = ck->layers[static_cast<size_t>(i)];
  if (name) *name = L.name.c_str();
  if (N) *N = L.N;
  if (K) *K = L.K;
  if (bits) *bits = L.bits;
  if (symmetric) *symmetric = L.symmetric ? 1 : 0;
  if (mask_len) *mask_len = static_cast<int64_t>(L.mask.size());
  if (rot_len) *rot_len = static_cast<int64_t>(L.rot.size());
  return DTQ_OK;
}

int dtq_checkpoint_load_layer(dtq_checkpoint_t ck, int64_t i, int act_bits, int hblock,
                              void* stream, dtq_qlinear_t* out) {
  NvtxRange nvtx_range("dtq_checkpoint_load_layer");
  if (!out) return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint_load_layer: null out");
  *out = nullptr;
  if (!ck || i < 0 || i >= static_cast<int64_t>(ck->layers.size()))
    return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint: bad layer index %lld", (long long)i);
  const CkptLayer& L = ck->layers[static_cast<size_t>(i)];
  // the GEMM's weight layout: symmetric, one group per output channel (Grouping 3)
  if (!L.symmetric || L.grouping != 3 || static_cast<int64_t>(L.scale.size()) != L.N)
    return fail(DTQ_ERR_UNSUPPORTED,
                "checkpoint layer '%s': only symmetric per-output-channel weights load "
                "onto the tensor-core GEMM", L.name.c_str());
  if (!L.mask.empty() && static_cast<int64_t>(L.mask.size()) != L.K)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint layer '%s': mask length != C_in",
                L.name.c_str());
  if (!L.rot.empty() && static_cast<int64_t>(L.rot.size()) != L.K)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "checkpoint layer '%s': rotation length != C_in",
                L.name.c_str());
  // the stored weights carry the full rot_len-point rotation (dtq_main.cpp
  // cmd_quantize: hadamard_matrix(w.cols())); the activations must get the
  // same one, never a block-diagonal one
  if (!L.rot.empty() && hblock != 0 && hblock != static_cast<int>(L.rot.size()))
    return fail(DTQ_ERR_INVALID_ARGUMENT,
                "checkpoint layer '%s': hblock %d differs from the stored rotation length %zu",
                L.name.c_str(), hblock, L.rot.size());
  DTQ_TRY(check_device());
  cudaStream_t st = as_stream(stream);
  std::vector<double> s(L.scale.begin(), L.scale.end());  // f32 -> f64, as read_checkpoint
  std::vector<double> smooth(L.mask.begin(), L.mask.end());
  uint8_t* d_codes = nullptr;
  double* d_s = nullptr;
  double* d_sm = nullptr;
  int8_t* d_rot = nullptr;
  int r = DTQ_OK;
  auto cleanup = [&] {
    if (d_codes) cudaFree(d_codes);
    if (d_s) cudaFree(d_s);
    if (d_sm) cudaFree(d_sm);
    if (d_rot) cudaFree(d_rot);
  };
  if (cudaMalloc(&d_codes, L.packed.size()) != cudaSuccess ||
      cudaMalloc(&d_s, s.size() * sizeof(double)) != cudaSuccess ||
      (!smooth.empty() && cudaMalloc(&d_sm, smooth.size() * sizeof(double)) != cudaSuccess) ||
      (!L.rot.empty() && cudaMalloc(&d_rot, L.rot.size()) != cudaSuccess)) {
    cleanup();
    return fail(DTQ_ERR_CUDA, "checkpoint_load_layer: out of device memory");
  }
  // the packed stream goes up as stored; the device unpacks it (W4: into the
  // GEMM's nibble layout, no host repack)
  if (cudaMemcpyAsync(d_codes, L.packed.data(), L.packed.size(), cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      cudaMemcpyAsync(d_s, s.data(), s.size() * sizeof(double), cudaMemcpyHostToDevice, st) !=
          cudaSuccess ||
      (d_sm && cudaMemcpyAsync(d_sm, smooth.data(), smooth.size() * sizeof(double),
                               cudaMemcpyHostToDevice, st) != cudaSuccess) ||
      (d_rot && cudaMemcpyAsync(d_rot, L.rot.data(), L.rot.size(), cudaMemcpyHostToDevice, st) !=
                    cudaSuccess)) {
    cleanup();
    return fail(DTQ_ERR_CUDA, "checkpoint_load_layer: upload failed");
  }
  dtq_balance bal{d_sm, d_rot, d_rot ? static_cast<int>(L.rot.size()) : 0};
  r = dtq_qlinear_create_from_codes(d_codes, 1, 0, L.bits, d_s, L.N, L.K, act_bits, nullptr,
                                    (d_sm || d_rot) ? &bal : nullptr, stream, out);
  if (cudaStreamSynchronize(st) != cudaSuccess && r == DTQ_OK)
    r = fail(DTQ_ERR_CUDA, "checkpoint_load_layer: device error");
  cleanup();
  return r;
}

// ------------------------------------------------------------------ mixed precision
int dtq_planned_create(const void* w, int w_dtype, int64_t N, int64_t K, int64_t ldw,
                       const int32_t* bits, int act_bits, const double* bias,
                       const dtq_balance* balance, void* stream, dtq_planned_t* out) {
  NvtxRange nvtx_range("dtq_planned_create");
  if (!out || !bits) return fail(DTQ_ERR_INVALID_ARGUMENT, "planned_create: null argument");
  *out = nullptr;
  for (int r = 0; r < kPlanRanges; ++r)
    if (!bits_supported(bits[r]))
      return fail(DTQ_ERR_INVALID_ARGUMENT,
                  "MixedPrecisionPlan: weight bits %d of range %d is not a quantized width "
                  "{2,4,6,8}", bits[r], r);
  auto* p = new dtq_planned_s();
  for (int r = 0; r < kPlanRanges; ++r) {
    p->bits[r] = bits[r];
    int have = -1;
    for (int q = 0; q < r; ++q)
      if (bits[q] == bits[r]) have = q;
    if (have >= 0) {
      p->range_handle[r] = p->range_handle[have];
      continue;
    }
    dtq_qlinear_t h = nullptr;
    const int st = dtq_qlinear_create(w, w_dtype, N, K, ldw, bits[r], act_bits, bias, balance,
                                      stream, &h);
    if (st != DTQ_OK) {
      dtq_planned_destroy(p);
      return st;
    }
    p->owned.push_back(h);
    p->range_handle[r] = h;
  }
  *out = p;
  return DTQ_OK;
}

int dtq_planned_destroy(dtq_planned_t p) {
  if (!p) return DTQ_OK;
  for (dtq_qlinear_t h : p->owned) dtq_qlinear_destroy(h);
  delete p;
  return DTQ_OK;
}

int dtq_planned_select(dtq_planned_t p, int64_t t, int64_t steps, dtq_qlinear_t* out) {
  if (!p || !out) return fail(DTQ_ERR_INVALID_ARGUMENT, "planned_select: null argument");
  if (steps <= 0 || t < 0 || t >= steps)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "planned_select: step %lld outside [0, %lld)",
                (long long)t, (long long)steps);
  *out = p->range_handle[t * kPlanRanges / steps];  // toydit.cpp:115
  return DTQ_OK;
}

int dtq_planned_bits(dtq_planned_t p, int r, int* bits) {
  if (!p || !bits || r < 0 || r >= kPlanRanges)
    return fail(DTQ_ERR_INVALID_ARGUMENT, "planned_bits: bad argument");
  *bits = p->bits[r];
  return DTQ_OK;
}

}  // extern "C"
