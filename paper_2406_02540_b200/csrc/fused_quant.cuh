// fused_quant.cuh -- the fused activation quantizer (FQ) for sm_100a.
//
// One HBM pass per token row:
//   load (128-bit, coalesced) -> [prologue: adaLN modulate | GELU | LN+modulate]
//   -> [smooth: X / s_c]                      (balance.cpp:57-67)
//   -> [blockwise Hadamard: signs, FWHT, 1/sqrt(hb)]  (balance.cpp:94-107 per block)
//   -> per-row min/max (or absmax) with warp shuffles + one smem hop
//   -> s, z in fp64 exactly as compute_minmax_params / compute_symmetric_params
//      (quant.cpp:90-124)
//   -> codes = clamp(round_half_even(v / s) + z, 0, 2^b - 1)   (quant.cpp:169-175)
//   -> u8 codes (64-bit stores), f64 scale, i32 zero point.
//
// Layout: a row of K elements is cut into 8-element "chunks"; thread t of
// the row's CTA owns chunks t, t + tpr, t + 2*tpr, ... (kCPT chunks).  A
// 128-column Hadamard block is therefore 16 consecutive lanes holding the
// same chunk index: butterflies with stride 1, 2, 4 stay in registers and
// strides 8..64 are __shfl_xor over lane masks 1..8.  Butterfly operands
// and order match the reference fwht exactly (a+b on the low index, a-b on
// the high one), so the fp64 "exact" instantiation is bit-identical to the
// reference rotate_channels.
//
// Arithmetic modes:
//   Tc = double ("exact"): every transform in fp64, divisions as in the
//     reference; codes, s and z are bit-identical to quantize() on the
//     same values, rotation and smoothing included.
//   Tc = float ("fast"): transforms in fp32; the quotient x/s is evaluated
//     as x * (float)(1/s) and only re-evaluated with an IEEE fp64 divide
//     when it lies within 2^-14 of a rounding tie, which bounds the fp32
//     error (|x/s| <= 255 => |err| <= 3.1e-5).  With no prologue, no
//     smoothing and no rotation the codes, s and z are therefore still
//     bit-identical to the reference for fp16/bf16/fp32 inputs.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "gelu.cuh"
#include "w4_unpack.cuh"

namespace dtq_fq {

enum Prologue : int { kProNone = 0, kProModulate = 1, kProGelu = 2, kProLnModulate = 3 };

struct FqArgs {
  const void* x;
  int64_t M, K, ldx;  // ldx in elements
  uint8_t* codes;
  int64_t ldc;        // bytes
  double* scale;
  int32_t* zero;
  int bits;
  int symmetric;
  const double* smooth_d;     // exact-mode divisor  (nullable)
  const float* inv_smooth_f;  // fast-mode multiplier (nullable)
  const int8_t* signs;        // rotation signs (nullable = no rotation)
  int hblock;
  const float* pro_scale;     // modulate: x*(1+scale)+shift
  const float* pro_shift;
  float eps;
  int32_t* status;            // nullable; |= 1 on non-finite input
  int pro;                    // Prologue
  int smooth_mul;             // 1: W * s (weight side of apply_scaling)
  const float* col_mul;       // fast kernel: folded sign/s_c/sqrt(hblock) per column
  int col_mul_const;          // 1: col_mul is a layer constant (written before the
                              // producer of X ran), readable before griddepcontrol.wait
  uint32_t* ready;            // tile kernel: per-128-row-block rows-ready counters the
                              // concurrently running GEMM waits on (nullptr: none)
  // host side (launcher only): the co-resident GEMM's per-SM registers and
  // shared memory; the launcher keeps `ready` only if one quantizer CTA fits
  // beside it on every SM, and reports that in *flags_used
  int partner_regs;
  int partner_smem;
  int* flags_used;
  unsigned long long* probe;  // diagnostics: per-warp phase cycles (or nullptr)
  int tpr;                    // threads per row (multiple of 16 and of hblock/8)
  int dbg;                    // diagnostics (tile kernel): 1 = skip the transform
  dtq_w4::Unpack w4;          // tile kernel: a W4A8 forward's weight expansion (w4_unpack.cuh)
  int* w4_done;               // launcher: 1 if the tile kernel took the w4 job
};

// ------------------------------------------------------------------ GELU
// (gelu.cuh: the same fp32 GELU is the GEMM's activation epilogue)
using dtq_act::gelu1;
using dtq_act::gelu2;

// ------------------------------------------------------------------ loads
template <typename T>
struct Vec;  // 8 elements in raw form
template <>
struct Vec<__half> {
  static constexpr int kWords = 1;  // uint4 words
};
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int kWords = 1;
};
template <>
struct Vec<float> {
  static constexpr int kWords = 2;
};
template <>
struct Vec<double> {
  static constexpr int kWords = 4;
};

template <typename Tin>
__device__ __forceinline__ void ld_raw(const Tin* p, uint4 (&r)[Vec<Tin>::kWords]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int w = 0; w < Vec<Tin>::kWords; ++w) r[w] = __ldcs(q + w);  // streaming: read once
}

template <typename Tc>
__device__ __forceinline__ void unpack(const uint4 (&r)[1], Tc (&v)[8], __half) {
  const __half2* h = reinterpret_cast<const __half2*>(&r[0]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(h[i]);
    v[2 * i] = static_cast<Tc>(f.x);
    v[2 * i + 1] = static_cast<Tc>(f.y);
  }
}
template <typename Tc>
__device__ __forceinline__ void unpack(const uint4 (&r)[1], Tc (&v)[8], __nv_bfloat16) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r[0]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h[i]);
    v[2 * i] = static_cast<Tc>(f.x);
    v[2 * i + 1] = static_cast<Tc>(f.y);
  }
}
template <typename Tc>
__device__ __forceinline__ void unpack(const uint4 (&r)[2], Tc (&v)[8], float) {
  const float* f = reinterpret_cast<const float*>(&r[0]);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = static_cast<Tc>(f[i]);
}
template <typename Tc>
__device__ __forceinline__ void unpack(const uint4 (&r)[4], Tc (&v)[8], double) {
  const double* f = reinterpret_cast<const double*>(&r[0]);
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = static_cast<Tc>(f[i]);
}

template <typename Tc, typename Tin>
__device__ __forceinline__ Tc to_c(Tin v) {
  return static_cast<Tc>(v);
}
template <>
__device__ __forceinline__ float to_c<float, __half>(__half v) {
  return __half2float(v);
}
template <>
__device__ __forceinline__ double to_c<double, __half>(__half v) {
  return static_cast<double>(__half2float(v));
}
template <>
__device__ __forceinline__ float to_c<float, __nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <>
__device__ __forceinline__ double to_c<double, __nv_bfloat16>(__nv_bfloat16 v) {
  return static_cast<double>(__bfloat162float(v));
}

// ------------------------------------------------------------------ reductions
template <typename T>
__device__ __forceinline__ T shfl_xor(T v, int m) {
  return __shfl_xor_sync(0xffffffffu, v, m);
}

// CTA-wide reduction of two values (a: min-like op, b: max-like op or sums).
// `buf` is a ping-pong smem area of 2 x 32 x 2 entries; one __syncthreads.
template <typename T, typename OpA, typename OpB>
__device__ __forceinline__ void block_reduce2(T& a, T& b, T* buf, int& pp, OpA opa, OpB opb) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    a = opa(a, shfl_xor(a, m));
    b = opb(b, shfl_xor(b, m));
  }
  const int nw = (blockDim.x + 31) >> 5;
  if (nw == 1) return;
  T* slot = buf + pp * 64;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    slot[2 * w] = a;
    slot[2 * w + 1] = b;
  }
  __syncthreads();
  a = slot[0];
  b = slot[1];
  for (int i = 1; i < nw; ++i) {
    a = opa(a, slot[2 * i]);
    b = opb(b, slot[2 * i + 1]);
  }
  pp ^= 1;
}

// ------------------------------------------------------------------ kernel
template <typename Tin, typename Tc, int kCPT, bool kVec>
__global__ void __launch_bounds__(kCPT == 1 ? 1024 : 256) fq_kernel(const FqArgs a) {
  constexpr bool kExact = sizeof(Tc) == 8;
  constexpr int kW = Vec<Tin>::kWords;
  // transform selection is uniform per launch: plain branches, no divergence
  const int kPro = a.pro;
  const bool kSmooth = a.smooth_d != nullptr || a.inv_smooth_f != nullptr;
  const bool kRotate = a.signs != nullptr;
  __shared__ __align__(16) Tc red[2 * 64];
  int pp = 0;

  const int t = threadIdx.x;
  const int tpr = a.tpr;
  const int K = static_cast<int>(a.K);
  const Tin* __restrict__ X = static_cast<const Tin*>(a.x);
  const int qmax_i = (1 << a.bits) - 1;

  // column base / valid count of each owned 8-element chunk.  With kVec the
  // host guarantees K % 8 == 0, so a chunk is either full or empty.
  int cb[kCPT], nv[kCPT];
#pragma unroll
  for (int i = 0; i < kCPT; ++i) {
    cb[i] = (i * tpr + t) * 8;
    const int rem = K - cb[i];
    nv[i] = t < tpr ? (rem >= 8 ? 8 : (rem > 0 ? rem : 0)) : 0;
  }
  auto ok = [&](int i, int e) -> bool { return kVec ? nv[i] > 0 : e < nv[i]; };

  // rotation signs stay in registers across rows (one bit per column);
  // smoothing / modulation vectors are re-read per row (L1-resident).
  uint32_t sgn[kCPT];
#pragma unroll
  for (int i = 0; i < kCPT; ++i) {
    sgn[i] = 0;
    if (kRotate)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (ok(i, e) && a.signs[cb[i] + e] < 0) sgn[i] |= 1u << e;
  }
  auto colvec = [&](const auto* p, int i, Tc (&out)[8], Tc fill) {
    if (kVec && nv[i] > 0) {
      if constexpr (sizeof(*p) == 4) {
        const float4 f0 = __ldg(reinterpret_cast<const float4*>(p + cb[i]));
        const float4 f1 = __ldg(reinterpret_cast<const float4*>(p + cb[i]) + 1);
        out[0] = f0.x; out[1] = f0.y; out[2] = f0.z; out[3] = f0.w;
        out[4] = f1.x; out[5] = f1.y; out[6] = f1.z; out[7] = f1.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; e += 2) {
          const double2 d = __ldg(reinterpret_cast<const double2*>(p + cb[i] + e));
          out[e] = static_cast<Tc>(d.x);
          out[e + 1] = static_cast<Tc>(d.y);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = e < nv[i] ? static_cast<Tc>(p[cb[i] + e]) : fill;
    }
  };

  uint4 raw[kCPT][kW];
  auto load_row = [&](int64_t row) {
    if constexpr (kVec) {
      const Tin* xr = X + row * a.ldx;
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
        if (nv[i] > 0) ld_raw<Tin>(xr + cb[i], raw[i]);
    }
  };

  int64_t row = blockIdx.x;
  if (row < a.M) load_row(row);
  for (; row < a.M; row += gridDim.x) {
    Tc v[kCPT][8];
    if constexpr (kVec) {
#pragma unroll
      for (int i = 0; i < kCPT; ++i) {
        if (nv[i] > 0) {
          unpack<Tc>(raw[i], v[i], Tin());
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[i][e] = Tc(0);
        }
      }
      const int64_t nxt = row + gridDim.x;
      if (nxt < a.M) load_row(nxt);  // prefetch the next row while this one is reduced
    } else {
      const Tin* xr = X + row * a.ldx;
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) v[i][e] = e < nv[i] ? to_c<Tc>(xr[cb[i] + e]) : Tc(0);
    }

    // non-finite guard (quant.cpp:143-146 throws std::invalid_argument)
    if (a.status != nullptr) {
      bool bad = false;
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) bad |= ok(i, e) && !isfinite(v[i][e]);
      if (bad) atomicOr(a.status, 1);
    }

    // ---- prologue (adaLN modulate, toydit.cpp:366-368; GELU toydit.cpp:83)
    if (kPro == kProLnModulate) {
      Tc s1 = 0, s2 = 0, dummy = 0;
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) s1 += ok(i, e) ? v[i][e] : Tc(0);
      block_reduce2(s1, dummy, red, pp, [](Tc p, Tc q) { return p + q; },
                    [](Tc p, Tc q) { return p + q; });
      const Tc mean = s1 / static_cast<Tc>(K);
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const Tc d = v[i][e] - mean;
          s2 += ok(i, e) ? d * d : Tc(0);
        }
      block_reduce2(s2, dummy, red, pp, [](Tc p, Tc q) { return p + q; },
                    [](Tc p, Tc q) { return p + q; });
      Tc rstd;
      if constexpr (kExact)
        rstd = 1.0 / sqrt(s2 / static_cast<double>(K) + static_cast<double>(a.eps));
      else
        rstd = rsqrtf(s2 / static_cast<float>(K) + a.eps);
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) v[i][e] = (v[i][e] - mean) * rstd;
    }
    if (kPro == kProModulate || kPro == kProLnModulate) {
#pragma unroll
      for (int i = 0; i < kCPT; ++i) {
        Tc sc[8], sh[8];
        colvec(a.pro_scale, i, sc, Tc(0));
        colvec(a.pro_shift, i, sh, Tc(0));
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if constexpr (kExact)  // no FMA contraction: reference rounds the product first
            v[i][e] = __dadd_rn(__dmul_rn(v[i][e], __dadd_rn(1.0, sc[e])), sh[e]);
          else
            v[i][e] = fmaf(v[i][e], 1.0f + sc[e], sh[e]);
        }
      }
    }
    if (kPro == kProGelu) {
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if constexpr (kExact)
            v[i][e] = 0.5 * v[i][e] * (1.0 + erf(v[i][e] / 1.4142135623730951));
          else
            v[i][e] = gelu1(static_cast<float>(v[i][e]));
        }
    }

    // ---- smoothing: X' = X / s_c (balance.cpp:62-63); W' = W * s_c on the weight side
    if (kSmooth) {
#pragma unroll
      for (int i = 0; i < kCPT; ++i) {
        Tc sm[8];
        if constexpr (kExact)
          colvec(a.smooth_d, i, sm, Tc(1));
        else
          colvec(a.inv_smooth_f, i, sm, Tc(1));
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (kExact && !a.smooth_mul)
            v[i][e] = v[i][e] / sm[e];
          else
            v[i][e] = v[i][e] * sm[e];
        }
      }
    }

    // ---- blockwise Hadamard (balance.cpp:94-107 per hblock columns)
    if (kRotate) {
#pragma unroll
      for (int i = 0; i < kCPT; ++i) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (sgn[i] & (1u << e)) v[i][e] = -v[i][e];
        // strides 1, 2, 4 inside the chunk (low index a+b, high index a-b)
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if ((e & h) == 0) {
              const Tc p = v[i][e], q = v[i][e + h];
              v[i][e] = p + q;
              v[i][e + h] = p - q;
            }
        // strides 8 .. hblock/2 across lanes: low lane v + o, high lane o - v,
        // both as one correctly rounded fma(+-1, v, o)
        for (int m = 1; m < (a.hblock >> 3); m <<= 1) {
          const Tc sg = (t & m) ? Tc(-1) : Tc(1);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const Tc o = shfl_xor(v[i][e], m);
            if constexpr (kExact)
              v[i][e] = fma(sg, v[i][e], o);
            else
              v[i][e] = fmaf(sg, v[i][e], o);
          }
        }
      }
      Tc norm;
      if constexpr (kExact)
        norm = 1.0 / sqrt(static_cast<double>(a.hblock));
      else
        norm = static_cast<float>(1.0 / sqrt(static_cast<double>(a.hblock)));
#pragma unroll
      for (int i = 0; i < kCPT; ++i)
#pragma unroll
        for (int e = 0; e < 8; ++e) v[i][e] *= norm;
    }

    // ---- per-row statistics
    Tc mn, mx;
    if constexpr (kExact) {
      mn = __longlong_as_double(0x7ff0000000000000LL);
    } else {
      mn = __int_as_float(0x7f800000);
    }
    mx = -mn;
#pragma unroll
    for (int i = 0; i < kCPT; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (ok(i, e)) {
          mn = fmin(mn, v[i][e]);
          mx = fmax(mx, v[i][e]);
        }
      }
    block_reduce2(mn, mx, red, pp, [](Tc p, Tc q) { return fmin(p, q); },
                  [](Tc p, Tc q) { return fmax(p, q); });

    // ---- params (quant.cpp:90-124), fp64 exactly as the reference
    const double qmax = static_cast<double>(qmax_i);
    const double dmn = static_cast<double>(mn), dmx = static_cast<double>(mx);
    double s, z;
    if (a.symmetric) {
      const double amax = fmax(fabs(dmn), fabs(dmx));
      z = static_cast<double>(1 << (a.bits - 1));
      s = amax > 0.0 ? amax / static_cast<double>((1 << (a.bits - 1)) - 1) : 1.0;
    } else if (dmx == dmn) {
      s = 1.0;
      z = fmin(fmax(rint(-dmn), 0.0), qmax);
    } else {
      const double lo = (0.0 < dmn) ? 0.0 : dmn;
      const double hi = (dmx < 0.0) ? 0.0 : dmx;
      s = (hi - lo) / qmax;
      z = fmin(fmax(rint(-lo / s), 0.0), qmax);
    }
    if (t == 0) {
      a.scale[row] = s;
      a.zero[row] = static_cast<int32_t>(z);
    }

    // ---- codes (quant.cpp:169-175): k = clamp(round_half_even(v / s) + z, 0, qmax)
    // q = v * (1/s) + z with one rounding; clamping before rounding is
    // equivalent (z is an integer).  Rounding-to-integer is the add of
    // 1.5 * 2^23 (fp32) or 1.5 * 2^52 (fp64), whose low bits are the code.
    // Quotients within the error bound of a .5 tie are redone with an
    // IEEE divide (rare, and warp-uniform per chunk).
    const double inv_s = 1.0 / s;
    uint8_t* crow = a.codes + row * a.ldc;
#pragma unroll
    for (int i = 0; i < kCPT; ++i) {
      if (nv[i] <= 0) continue;
      uint32_t m[8];
      bool near = false;
      if constexpr (kExact) {
        const double zq = z, qq = qmax;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double q = fmin(fmax(fma(v[i][e], inv_s, zq), 0.0), qq);
          const double r = q + 6755399441055744.0;  // 1.5 * 2^52
          near |= fabs(q - (r - 6755399441055744.0)) > 0.5 - 1e-9;
          m[e] = static_cast<uint32_t>(__double2loint(r));
        }
      } else {
        const float inv_sf = static_cast<float>(inv_s), zf = static_cast<float>(z);
        const float qf = static_cast<float>(qmax_i);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float q = fminf(fmaxf(fmaf(v[i][e], inv_sf, zf), 0.f), qf);
          const float r = q + 12582912.0f;  // 1.5 * 2^23
          near |= fabsf(q - (r - 12582912.0f)) > 0.5f - 6.103515625e-05f;
          m[e] = __float_as_uint(r);
        }
      }
      if (near) {
        // exact re-evaluation of the near-tie quotients (fp64 IEEE divide)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double k = fmin(fmax(rint(static_cast<double>(v[i][e]) / s) + z, 0.0), qmax);
          m[e] = static_cast<uint32_t>(k);
        }
      }
      const uint32_t p0 = __byte_perm(__byte_perm(m[0], m[1], 0x0040), __byte_perm(m[2], m[3], 0x0040), 0x5410);
      const uint32_t p1 = __byte_perm(__byte_perm(m[4], m[5], 0x0040), __byte_perm(m[6], m[7], 0x0040), 0x5410);
      uint8_t* dst = crow + cb[i];
      if (kVec) {
        *reinterpret_cast<uint2*>(dst) = make_uint2(p0, p1);
      } else {
        for (int e = 0; e < nv[i]; ++e) dst[e] = static_cast<uint8_t>((e < 4 ? p0 : p1) >> (8 * (e & 3)));
      }
    }
  }
}

}  // namespace dtq_fq
