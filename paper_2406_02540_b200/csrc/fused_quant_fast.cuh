// fused_quant_fast.cuh -- fp32 ("fast") fused quantizer.
//
// Same contract as fq_kernel (fused_quant.cuh) with fp32 transforms, built
// for throughput on a memory-bound op:
//   * one warp per token row, any K.  The whole input row arrives by one
//     bulk async copy (cp.async.bulk, mbarrier-completed) into a per-warp
//     double buffer, issued one row AHEAD, so HBM latency overlaps the
//     previous row's arithmetic; the row is then walked in 256-column steps
//     from shared memory and the transformed fp32 values parked in a per-warp
//     row buffer: registers stay low and the loop body is small;
//   * sign flip, smoothing (1/s_c) and the 1/sqrt(128) normalisation are one
//     folded per-column multiplier (col_mul, L1-resident) applied before the
//     butterflies (linearity; differs from the fp64 reference only by
//     rounding, covered by the 1-LSB parity bar);
//   * 128-column Walsh-Hadamard butterflies: strides 1/2/4 in registers
//     (packed FADD2), strides 8..64 via __shfl_xor within 16-lane groups;
//   * codes: q = v*(1/s)+z in one FFMA2, rounding by the 1.5*2^23 add whose
//     low byte is the code; |frac - 1/2| < 2^-14 (the fp32 error bound) is
//     recomputed with an IEEE fp64 divide (rare); the clamp is skipped on
//     rows whose min-max params already bound q (the bounds themselves are
//     near-ties and take the exact path).
// With no prologue, smoothing or rotation the codes, s and z are
// bit-identical to the reference (quant.cpp:90-113, 169-175).
// Host contract: K % 8 == 0, 16-byte aligned rows, rotation block 128,
// dynamic smem = fq_fast_smem_bytes(warps_per_cta, K, sizeof(Tin)).
#pragma once

#include "fused_quant.cuh"
#include "ptx.cuh"

namespace dtq_fq {

__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  return __ffma2_rn(b, make_float2(-1.f, -1.f), a);
}

// per warp: 2 raw input rows (K * sizeof(Tin), 128-byte padded), the fp32 row
// buffer (ceil(K/256) KB) and 2 mbarriers
__host__ __device__ constexpr size_t fq_fast_warp_bytes(int64_t K, int in_bytes) {
  return 2 * ((static_cast<size_t>(K) * in_bytes + 127) / 128 * 128) +
         static_cast<size_t>((K + 255) / 256) * 1024 + 16;
}
__host__ __device__ constexpr size_t fq_fast_smem_bytes(int warps, int64_t K, int in_bytes) {
  return static_cast<size_t>(warps) * fq_fast_warp_bytes(K, in_bytes);
}

template <typename Tin>
__device__ __forceinline__ void load8(const Tin* p, bool ok, float (&v)[8]) {  // shared memory
  uint4 r[Vec<Tin>::kWords];
#pragma unroll
  for (int w = 0; w < Vec<Tin>::kWords; ++w)
    r[w] = ok ? reinterpret_cast<const uint4*>(p)[w] : make_uint4(0u, 0u, 0u, 0u);
  unpack<float>(r, v, Tin());
}

// kNit > 0: the row has exactly kNit 256-column steps (compile-time; one warp
// per row, fully unrolled, only the last step can be partial); kNit == 0:
// runtime step count, W = tpr/32 warps per row.
template <typename Tin, bool kRot, int kNit>
__global__ void __launch_bounds__(256) fq_fast_kernel(const FqArgs a) {
  extern __shared__ __align__(128) uint8_t fq_smem[];
  const int lane = threadIdx.x & 31;
  const int W = kNit > 0 ? 1 : (a.tpr >> 5);  // warps per row group
  const int g = (threadIdx.x >> 5) / W;      // row group in the CTA
  const int wg = (threadIdx.x >> 5) - g * W; // warp within the group
  const int groups = (blockDim.x >> 5) / W;
  const int K = static_cast<int>(a.K);
  const int chunks = K >> 3;
  const int nit = kNit > 0 ? kNit : (chunks + 31) >> 5;  // 256-column steps (step i -> warp i % W)
  const uint32_t row_in = static_cast<uint32_t>(K) * sizeof(Tin);
  const size_t raw_pitch = (static_cast<size_t>(row_in) + 127) / 128 * 128;
  uint8_t* wbase = fq_smem + g * fq_fast_warp_bytes(K, sizeof(Tin));
  uint8_t* const raw0 = wbase;
  uint8_t* const raw1 = wbase + raw_pitch;
  float* buf = reinterpret_cast<float*>(wbase + 2 * raw_pitch);  // [step][half][lane][4]
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + 2 * raw_pitch + nit * 1024);
  __shared__ float red[8][4][2];  // [group][warp][min, max]
  const Tin* __restrict__ X = static_cast<const Tin*>(a.x);
  const int qmax_i = (1 << a.bits) - 1;
  const float sg_1 = (lane & 1) ? -1.f : 1.f, sg_2 = (lane & 2) ? -1.f : 1.f;
  const float sg_4 = (lane & 4) ? -1.f : 1.f, sg_8 = (lane & 8) ? -1.f : 1.f;
  const bool leader = wg == 0 && lane == 0;  // issues the group's row copies
  auto group_sync = [&]() {
    if (W > 1)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(32 * W) : "memory");
    else
      __syncwarp();
  };

  if (leader) {
    dtq_ptx::mbar_init(&bar[0], 1);
    dtq_ptx::mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t rstep = static_cast<int64_t>(gridDim.x) * groups;
  auto issue = [&](int64_t r, int b) {  // leader: bulk copy of row r into raw[b]
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of raw[b]
    dtq_ptx::mbar_arrive_expect_tx(&bar[b], row_in);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            dtq_ptx::smem_u32(b ? raw1 : raw0)),
        "l"(reinterpret_cast<uint64_t>(X + r * a.ldx)), "r"(row_in), "r"(dtq_ptx::smem_u32(&bar[b]))
        : "memory");
  };
  int64_t row = static_cast<int64_t>(blockIdx.x) * groups + g;
  if (leader && row < a.M) issue(row, 0);
  uint32_t phase = 0u;  // bit b = parity of bar[b]

  for (int it = 0; row < a.M; row += rstep, ++it) {
    const int b = it & 1;
    if (leader && row + rstep < a.M) issue(row + rstep, b ^ 1);  // next row, in flight now
    long long tp0 = a.probe ? clock64() : 0;
    dtq_ptx::mbar_wait(&bar[b], (phase >> b) & 1u);
    long long tp1 = a.probe ? clock64() : 0;
    phase ^= 1u << b;
    const Tin* xr = reinterpret_cast<const Tin*>(b ? raw1 : raw0);  // this row, in smem

    // ---- optional LayerNorm statistics (extra pass over the row, L1/L2 hits)
    float mean = 0.f, rstd = 1.f;
    if (a.pro == kProLnModulate) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll(kNit > 0 ? kNit : 1)
      for (int i = wg; i < nit; i += W) {
        const int c = i * 32 + lane;
        float v[8];
        load8<Tin>(xr + c * 8, (kNit > 0 && i < kNit - 1) || c < chunks, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) s1 += v[e];
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, m);
      if (W > 1) {
        if (lane == 0) red[g][wg][0] = s1;
        group_sync();
        s1 = 0.f;
        for (int w = 0; w < W; ++w) s1 += red[g][w][0];
        group_sync();
      }
      mean = s1 / static_cast<float>(K);
#pragma unroll(kNit > 0 ? kNit : 1)
      for (int i = wg; i < nit; i += W) {
        const int c = i * 32 + lane;
        const bool ok = (kNit > 0 && i < kNit - 1) || c < chunks;
        float v[8];
        load8<Tin>(xr + c * 8, ok, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) s2 += ok ? (v[e] - mean) * (v[e] - mean) : 0.f;
      }
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, m);
      if (W > 1) {
        if (lane == 0) red[g][wg][0] = s2;
        group_sync();
        s2 = 0.f;
        for (int w = 0; w < W; ++w) s2 += red[g][w][0];
        group_sync();
      }
      rstd = rsqrtf(s2 / static_cast<float>(K) + a.eps);
    }

    // ---- pass 1: load, prologue, multiplier, butterflies, min / max -> smem
    float mn = __int_as_float(0x7f800000), mx = -mn;
    bool bad = false;
#pragma unroll(kNit > 0 ? kNit : 1)
    for (int i = wg; i < nit; i += W) {
      const int c = i * 32 + lane;
      const bool ok = (kNit > 0 && i < kNit - 1) || c < chunks;
      float v[8];
      load8<Tin>(xr + c * 8, ok, v);
      if (a.status != nullptr) {
#pragma unroll
        for (int e = 0; e < 8; ++e) bad |= ok && !isfinite(v[e]);
      }
      if (a.pro != kProNone) {
        if (a.pro == kProGelu) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] = 0.5f * v[e] * (1.0f + erff(v[e] * 0.70710678118654752f));
        } else if (ok) {
          if (a.pro == kProLnModulate) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = (v[e] - mean) * rstd;
          }
          const float4 c0 = __ldg(reinterpret_cast<const float4*>(a.pro_scale + c * 8));
          const float4 c1 = __ldg(reinterpret_cast<const float4*>(a.pro_scale + c * 8) + 1);
          const float4 h0 = __ldg(reinterpret_cast<const float4*>(a.pro_shift + c * 8));
          const float4 h1 = __ldg(reinterpret_cast<const float4*>(a.pro_shift + c * 8) + 1);
          const float sc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
          const float sh[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = fmaf(v[e], 1.0f + sc[e], sh[e]);
        }
      }
      if (a.col_mul != nullptr) {
        const int cc = ok ? c : 0;
        const float4 m0 = __ldg(reinterpret_cast<const float4*>(a.col_mul + cc * 8));
        const float4 m1 = __ldg(reinterpret_cast<const float4*>(a.col_mul + cc * 8) + 1);
        const float2 r0 = __fmul2_rn(make_float2(v[0], v[1]), make_float2(m0.x, m0.y));
        const float2 r1 = __fmul2_rn(make_float2(v[2], v[3]), make_float2(m0.z, m0.w));
        const float2 r2 = __fmul2_rn(make_float2(v[4], v[5]), make_float2(m1.x, m1.y));
        const float2 r3 = __fmul2_rn(make_float2(v[6], v[7]), make_float2(m1.z, m1.w));
        v[0] = r0.x; v[1] = r0.y; v[2] = r1.x; v[3] = r1.y;
        v[4] = r2.x; v[5] = r2.y; v[6] = r3.x; v[7] = r3.y;
      }
      if constexpr (kRot) {
        // strides 1, 2 (packed pairs P_k = (v_k, v_k+4)) and 4 in registers
        float2 P0 = make_float2(v[0], v[4]), P1 = make_float2(v[1], v[5]);
        float2 P2 = make_float2(v[2], v[6]), P3 = make_float2(v[3], v[7]);
        float2 t0 = f2add(P0, P1), t1 = f2sub(P0, P1), t2 = f2add(P2, P3), t3 = f2sub(P2, P3);
        P0 = f2add(t0, t2); P2 = f2sub(t0, t2); P1 = f2add(t1, t3); P3 = f2sub(t1, t3);
        v[0] = P0.x + P0.y; v[4] = P0.x - P0.y;
        v[1] = P1.x + P1.y; v[5] = P1.x - P1.y;
        v[2] = P2.x + P2.y; v[6] = P2.x - P2.y;
        v[3] = P3.x + P3.y; v[7] = P3.x - P3.y;
        // strides 8, 16, 32, 64: lanes xor 1, 2, 4, 8 (low lane v + o, high o - v)
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const int m = 1 << st;
          const float sg = st == 0 ? sg_1 : (st == 1 ? sg_2 : (st == 2 ? sg_4 : sg_8));
          const float2 sg2 = make_float2(sg, sg);
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const float o0 = __shfl_xor_sync(0xffffffffu, v[e], m);
            const float o1 = __shfl_xor_sync(0xffffffffu, v[e + 1], m);
            const float2 r = __ffma2_rn(sg2, make_float2(v[e], v[e + 1]), make_float2(o0, o1));
            v[e] = r.x;
            v[e + 1] = r.y;
          }
        }
      }
      if (ok) {
        float cmn = fminf(fminf(fminf(v[0], v[1]), fminf(v[2], v[3])),
                          fminf(fminf(v[4], v[5]), fminf(v[6], v[7])));
        float cmx = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])),
                          fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
        mn = fminf(mn, cmn);
        mx = fmaxf(mx, cmx);
      }
      float* bp = buf + i * 256 + lane * 4;
      *reinterpret_cast<float4*>(bp) = make_float4(v[0], v[1], v[2], v[3]);
      *reinterpret_cast<float4*>(bp + 128) = make_float4(v[4], v[5], v[6], v[7]);
    }
    if (bad) atomicOr(a.status, 1);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, m));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    }
    if (W > 1) {
      if (lane == 0) {
        red[g][wg][0] = mn;
        red[g][wg][1] = mx;
      }
      group_sync();
      for (int w = 0; w < W; ++w) {
        mn = fminf(mn, red[g][w][0]);
        mx = fmaxf(mx, red[g][w][1]);
      }
    }

    long long tp2 = a.probe ? clock64() : 0;
    // ---- params (quant.cpp:90-124) in fp64 exactly as the reference
    const double qmax = static_cast<double>(qmax_i);
    const double dmn = static_cast<double>(mn), dmx = static_cast<double>(mx);
    double s, z;
    bool need_clamp = a.symmetric || a.bits != 8;
    if (a.symmetric) {
      const double amax = fmax(fabs(dmn), fabs(dmx));
      z = static_cast<double>(1 << (a.bits - 1));
      s = amax > 0.0 ? amax / static_cast<double>((1 << (a.bits - 1)) - 1) : 1.0;
    } else if (dmx == dmn) {
      s = 1.0;
      z = fmin(fmax(rint(-dmn), 0.0), qmax);
      need_clamp = true;
    } else {
      const double lo = (0.0 < dmn) ? 0.0 : dmn;
      const double hi = (dmx < 0.0) ? 0.0 : dmx;
      s = (hi - lo) / qmax;
      z = fmin(fmax(rint(-lo / s), 0.0), qmax);
    }
    if (leader) {
      a.scale[row] = s;
      a.zero[row] = static_cast<int32_t>(z);
    }

    long long tp3 = a.probe ? clock64() : 0;
    // ---- pass 2: codes from the parked values
    const float inv_sf = static_cast<float>(1.0 / s), zf = static_cast<float>(z);
    const float qf = static_cast<float>(qmax_i);
    const float2 inv2 = make_float2(inv_sf, inv_sf), z2 = make_float2(zf, zf);
    const float2 mg2 = make_float2(12582912.0f, 12582912.0f);
    const float2 nmg2 = make_float2(-12582912.0f, -12582912.0f);
    uint8_t* crow = a.codes + row * a.ldc;
#pragma unroll(kNit > 0 ? kNit : 1)
    for (int i = wg; i < nit; i += W) {
      const int c = i * 32 + lane;
      if (!((kNit > 0 && i < kNit - 1) || c < chunks)) continue;
      const float* bp = buf + i * 256 + lane * 4;
      const float4 a0 = *reinterpret_cast<const float4*>(bp);
      const float4 a1 = *reinterpret_cast<const float4*>(bp + 128);
      const float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      uint32_t m[8];
      float dm = 0.f;
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float2 q = __ffma2_rn(make_float2(v[e], v[e + 1]), inv2, z2);
        if (need_clamp) {
          q.x = fminf(fmaxf(q.x, 0.f), qf);
          q.y = fminf(fmaxf(q.y, 0.f), qf);
        }
        const float2 r = __fadd2_rn(q, mg2);             // round to the integer code
        const float2 d = f2sub(q, __fadd2_rn(r, nmg2));  // q - round(q), exact
        dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
        m[e] = __float_as_uint(r.x);
        m[e + 1] = __float_as_uint(r.y);
      }
      if (dm > 0.5f - 6.103515625e-05f) {
        // within the fp32 error bound of a .5 tie: exact fp64 re-evaluation
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double k = fmin(fmax(rint(static_cast<double>(v[e]) / s) + z, 0.0), qmax);
          m[e] = static_cast<uint32_t>(k);
        }
      }
      const uint32_t p0 = __byte_perm(__byte_perm(m[0], m[1], 0x0040), __byte_perm(m[2], m[3], 0x0040), 0x5410);
      const uint32_t p1 = __byte_perm(__byte_perm(m[4], m[5], 0x0040), __byte_perm(m[6], m[7], 0x0040), 0x5410);
      *reinterpret_cast<uint2*>(crow + c * 8) = make_uint2(p0, p1);
    }
    group_sync();  // the whole group is done with this raw buffer (and red) before reuse
    if (a.probe && lane == 0) {
      const long long tp4 = clock64();
      unsigned long long* pr = a.probe + 8 * ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
      pr[0] += tp1 - tp0;  // wait for the row copy
      pr[1] += tp2 - tp1;  // pass 1 (+ reduce)
      pr[2] += tp3 - tp2;  // params
      pr[3] += tp4 - tp3;  // pass 2 + group sync
      pr[4] += 1;          // rows
    }
  }
}

}  // namespace dtq_fq
