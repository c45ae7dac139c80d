// fused_quant_fast.cuh -- fp32 ("fast") fused quantizer.
//
// Same contract as fq_kernel (fused_quant.cuh) with fp32 transforms, built
// for throughput on a memory-bound op.
//
// Work decomposition.  A 128-column block of a row is owned by an 8-lane
// group, 16 consecutive columns per lane (two 128-bit loads, one 128-bit
// code store).  A warp = 4 lane groups; G = 1, 2 or 4 groups cooperate on a
// row, so one warp holds R = 4/G rows at once and walks their blocks in
// nblocks/G steps.  Consequences:
//   * the 128-point Walsh-Hadamard transform needs 4 in-register stages
//     (strides 1..8, three of them packed FADD2/FFMA2) and only 3 shuffle
//     stages (strides 16, 32, 64 = lane xor 1, 2, 4);
//   * the fp64 parameter math (quant.cpp:90-113) runs once per warp for R
//     rows at a time;
//   * row min/max = 3 + log2(G) shuffle levels, no barriers.
// Input rows arrive by one bulk async copy per row (cp.async.bulk,
// mbarrier-completed) into shared memory; the next row group is fetched as
// soon as pass 1 has consumed the current one, overlapping the parameter
// math and the code pass.  Transformed values are parked in a per-warp fp32
// row buffer between the min/max pass and the code pass.
//
// Arithmetic.  Sign flip, smoothing (1/s_c) and 1/sqrt(128) are ONE folded
// per-column multiplier (col_mul) applied before the butterflies (linearity;
// differs from the fp64 reference only by rounding, within the 1-LSB parity
// bar).  Codes: q = v*(1/s)+z in one FFMA2, rounding by the 1.5*2^23 add
// whose low byte is the code; |frac - 1/2| < 2^-14 (the fp32 error bound)
// is recomputed with an IEEE fp64 divide (rare); the clamp is skipped on rows
// whose min-max params already bound q (those bounds are near-ties and take
// the exact path).  With no prologue, smoothing or rotation the codes, s and
// z are bit-identical to the reference (quant.cpp:90-113, 169-175).
//
// Host contract: K % 128 == 0, 16-byte aligned rows, rotation block 128,
// blockDim = 32 * warps, dynamic smem = warps * fq_fast_warp_bytes(K, G, in).
#pragma once

#include "fused_quant.cuh"
#include "ptx.cuh"

namespace dtq_fq {

__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  return __ffma2_rn(b, make_float2(-1.f, -1.f), a);
}

// per warp: R = 4/G raw input rows + R fp32 rows + 1 mbarrier
__host__ __device__ constexpr size_t fq_fast_warp_bytes(int64_t K, int G, int in_bytes) {
  return static_cast<size_t>(4 / G) * static_cast<size_t>(K) * (in_bytes + 4) + 16;
}

template <typename Tin>
__device__ __forceinline__ void load16(const Tin* p, float (&v)[16]) {  // shared memory
  uint4 r0[Vec<Tin>::kWords], r1[Vec<Tin>::kWords];
#pragma unroll
  for (int w = 0; w < Vec<Tin>::kWords; ++w) {
    r0[w] = reinterpret_cast<const uint4*>(p)[w];
    r1[w] = reinterpret_cast<const uint4*>(p + 8)[w];
  }
  float a[8], b[8];
  unpack<float>(r0, a, Tin());
  unpack<float>(r1, b, Tin());
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    v[e] = a[e];
    v[e + 8] = b[e];
  }
}

// kNblk > 0: compile-time K = 128 * kNblk (static steps, offsets and
// predicates); kNblk == 0: runtime K.
template <typename Tin, bool kRot, int G, int kNblk>
__global__ void __launch_bounds__(256) fq_fast_kernel(const FqArgs a) {
  constexpr int R = 4 / G;  // rows per warp
  extern __shared__ __align__(128) uint8_t fq_smem[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int lg = lane >> 3;  // lane group 0..3
  const int li = lane & 7;   // lane within the group
  const int rl = lg / G;     // local row of this lane group
  const int gi = lg % G;     // group index within the row
  const int K = kNblk > 0 ? 128 * kNblk : static_cast<int>(a.K);
  const int nblk = K >> 7;
  const int steps = (nblk + G - 1) / G;
  // block st*G+gi is valid for every lane group except possibly in the last step
  auto blk_ok = [&](int st, int blk) -> bool {
    return (kNblk > 0 && (st + 1) * G <= kNblk) || blk < nblk;
  };
  uint8_t* wbase = fq_smem + warp * fq_fast_warp_bytes(K, G, sizeof(Tin));
  const Tin* raw = reinterpret_cast<const Tin*>(wbase);  // [R][K]
  float* park = reinterpret_cast<float*>(wbase + static_cast<size_t>(R) * K * sizeof(Tin));
  uint64_t* bar =
      reinterpret_cast<uint64_t*>(wbase + static_cast<size_t>(R) * K * (sizeof(Tin) + 4));
  const Tin* __restrict__ X = static_cast<const Tin*>(a.x);
  const int qmax_i = (1 << a.bits) - 1;
  const uint32_t row_in = static_cast<uint32_t>(K) * sizeof(Tin);
  const float sgn1 = (li & 1) ? -1.f : 1.f, sgn2 = (li & 2) ? -1.f : 1.f;
  const float sgn4 = (li & 4) ? -1.f : 1.f;

  if (lane == 0) {
    dtq_ptx::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t gstride = static_cast<int64_t>(gridDim.x) * nwarps * R;
  // lane 0 fetches the R rows of a group (rows past M are skipped)
  auto issue = [&](int64_t g0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    int n = 0;
    for (int r = 0; r < R; ++r) n += (g0 + r < a.M) ? 1 : 0;
    dtq_ptx::mbar_arrive_expect_tx(bar, row_in * n);
    for (int r = 0; r < n; ++r)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(dtq_ptx::smem_u32(raw + static_cast<size_t>(r) * K)),
          "l"(reinterpret_cast<uint64_t>(X + (g0 + r) * a.ldx)), "r"(row_in),
          "r"(dtq_ptx::smem_u32(bar))
          : "memory");
  };
  int64_t r0 = (static_cast<int64_t>(blockIdx.x) * nwarps + warp) * R;
  if (lane == 0 && r0 < a.M) issue(r0);
  uint32_t phase = 0;

  for (; r0 < a.M; r0 += gstride) {
    const int64_t row = r0 + rl;
    const bool row_ok = row < a.M;
    dtq_ptx::mbar_wait(bar, phase);
    phase ^= 1u;
    const Tin* xr = raw + static_cast<size_t>(rl) * K;
    float* pr = park + static_cast<size_t>(rl) * K;  // [block][quarter][lane][4]

    // ---- optional LayerNorm statistics (reads the row from smem)
    float mean = 0.f, rstd = 1.f;
    if (a.pro == kProLnModulate) {
      float s1 = 0.f, s2 = 0.f;
      for (int st = 0; st < steps; ++st) {
        const int blk = st * G + gi;
        if (row_ok && blk < nblk) {
          float v[16];
          load16<Tin>(xr + blk * 128 + li * 16, v);
#pragma unroll
          for (int e = 0; e < 16; ++e) s1 += v[e];
        }
      }
#pragma unroll
      for (int m = 1; m < 8 * G; m <<= 1) s1 += __shfl_xor_sync(0xffffffffu, s1, m);
      mean = s1 / static_cast<float>(K);
      for (int st = 0; st < steps; ++st) {
        const int blk = st * G + gi;
        if (row_ok && blk < nblk) {
          float v[16];
          load16<Tin>(xr + blk * 128 + li * 16, v);
#pragma unroll
          for (int e = 0; e < 16; ++e) s2 += (v[e] - mean) * (v[e] - mean);
        }
      }
#pragma unroll
      for (int m = 1; m < 8 * G; m <<= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, m);
      rstd = rsqrtf(s2 / static_cast<float>(K) + a.eps);
    }

    // ---- pass 1: prologue, multiplier, butterflies, min / max; park in smem
    float mn = __int_as_float(0x7f800000), mx = -mn;
    bool bad = false;
#pragma unroll(kNblk > 0 ? (kNblk + G - 1) / G : 1)
    for (int st = 0; st < steps; ++st) {
      const int blk = st * G + gi;
      const bool ok = row_ok && blk_ok(st, blk);
      const int c0 = (ok ? blk : 0) * 128 + li * 16;  // first column of this lane
      float v[16];
      if (ok) {
        load16<Tin>(xr + c0, v);
      } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = 0.f;
      }
      if (a.status != nullptr) {
#pragma unroll
        for (int e = 0; e < 16; ++e) bad |= ok && !isfinite(v[e]);
      }
      if (a.pro != kProNone) {
        if (a.pro == kProGelu) {
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float2 g = gelu2(make_float2(v[e], v[e + 1]));
            v[e] = g.x;
            v[e + 1] = g.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 sc = __ldg(reinterpret_cast<const float4*>(a.pro_scale + c0) + q);
            const float4 sh = __ldg(reinterpret_cast<const float4*>(a.pro_shift + c0) + q);
            const float scv[4] = {sc.x, sc.y, sc.z, sc.w}, shv[4] = {sh.x, sh.y, sh.z, sh.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              float x = v[4 * q + u];
              if (a.pro == kProLnModulate) x = (x - mean) * rstd;
              v[4 * q + u] = fmaf(x, 1.0f + scv[u], shv[u]);
            }
          }
        }
      }
      if (a.col_mul != nullptr) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 m = __ldg(reinterpret_cast<const float4*>(a.col_mul + c0) + q);
          const float2 p0 = __fmul2_rn(make_float2(v[4 * q], v[4 * q + 1]), make_float2(m.x, m.y));
          const float2 p1 =
              __fmul2_rn(make_float2(v[4 * q + 2], v[4 * q + 3]), make_float2(m.z, m.w));
          v[4 * q] = p0.x;
          v[4 * q + 1] = p0.y;
          v[4 * q + 2] = p1.x;
          v[4 * q + 3] = p1.y;
        }
      }
      if constexpr (kRot) {
        // pairs P_k = (v_k, v_k+8): strides 1, 2, 4 are packed butterflies
        float2 P[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) P[k] = make_float2(v[k], v[k + 8]);
#pragma unroll
        for (int h = 1; h < 8; h <<= 1)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if ((k & h) == 0) {
              const float2 sm = f2add(P[k], P[k + h]), df = f2sub(P[k], P[k + h]);
              P[k] = sm;
              P[k + h] = df;
            }
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // stride 8: within each pair
          v[k] = P[k].x + P[k].y;
          v[k + 8] = P[k].x - P[k].y;
        }
        // strides 16, 32, 64: lanes xor 1, 2, 4 (low lane v + o, high lane o - v)
#pragma unroll
        for (int s3 = 0; s3 < 3; ++s3) {
          const int m = 1 << s3;
          const float sg = s3 == 0 ? sgn1 : (s3 == 1 ? sgn2 : sgn4);
          const float2 sg2 = make_float2(sg, sg);
#pragma unroll
          for (int e = 0; e < 16; e += 2) {
            const float o0 = __shfl_xor_sync(0xffffffffu, v[e], m);
            const float o1 = __shfl_xor_sync(0xffffffffu, v[e + 1], m);
            const float2 r = __ffma2_rn(sg2, make_float2(v[e], v[e + 1]), make_float2(o0, o1));
            v[e] = r.x;
            v[e + 1] = r.y;
          }
        }
      }
      if (ok) {
        float cmn = fminf(v[0], v[15]), cmx = fmaxf(v[0], v[15]);
#pragma unroll
        for (int e = 1; e < 15; e += 2) {
          cmn = fminf(cmn, fminf(v[e], v[e + 1]));
          cmx = fmaxf(cmx, fmaxf(v[e], v[e + 1]));
        }
        mn = fminf(mn, cmn);
        mx = fmaxf(mx, cmx);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(pr + (blk * 4 + q) * 32 + li * 4) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
    if (bad) atomicOr(a.status, 1);
    __syncwarp();
    // the raw rows are consumed: fetch the next group while params and codes run
    if (lane == 0 && r0 + gstride < a.M) issue(r0 + gstride);
#pragma unroll
    for (int m = 1; m < 8 * G; m <<= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, m));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, m));
    }

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
    if (row_ok && gi == 0 && li == 0) {
      a.scale[row] = s;
      a.zero[row] = static_cast<int32_t>(z);
    }

    // ---- pass 2: codes from the parked values, 16 per lane -> one 128-bit store
    const float inv_sf = static_cast<float>(1.0 / s), zf = static_cast<float>(z);
    const float qf = static_cast<float>(qmax_i);
    const float2 inv2 = make_float2(inv_sf, inv_sf), z2 = make_float2(zf, zf);
    const float2 mg2 = make_float2(12582912.0f, 12582912.0f);
    const float2 nmg2 = make_float2(-12582912.0f, -12582912.0f);
    uint8_t* crow = a.codes + row * a.ldc;
#pragma unroll(kNblk > 0 ? (kNblk + G - 1) / G : 1)
    for (int st = 0; st < steps; ++st) {
      const int blk = st * G + gi;
      if (!(row_ok && blk_ok(st, blk))) continue;
      float v[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 t = *reinterpret_cast<const float4*>(pr + (blk * 4 + q) * 32 + li * 4);
        v[4 * q] = t.x;
        v[4 * q + 1] = t.y;
        v[4 * q + 2] = t.z;
        v[4 * q + 3] = t.w;
      }
      uint32_t mq[16];
      float dm = 0.f;
#pragma unroll
      for (int e = 0; e < 16; e += 2) {
        float2 q = __ffma2_rn(make_float2(v[e], v[e + 1]), inv2, z2);
        if (need_clamp) {
          q.x = fminf(fmaxf(q.x, 0.f), qf);
          q.y = fminf(fmaxf(q.y, 0.f), qf);
        }
        const float2 r = __fadd2_rn(q, mg2);             // round to the integer code
        const float2 d = f2sub(q, __fadd2_rn(r, nmg2));  // q - round(q), exact
        dm = fmaxf(dm, fmaxf(fabsf(d.x), fabsf(d.y)));
        mq[e] = __float_as_uint(r.x);
        mq[e + 1] = __float_as_uint(r.y);
      }
      if (dm > 0.5f - 6.103515625e-05f) {
        // within the fp32 error bound of a .5 tie: exact fp64 re-evaluation of
        // just those elements (a warp pays for element e only if a lane needs it)
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float2 q = __ffma2_rn(make_float2(v[e], v[e]), inv2, z2);
          if (need_clamp) q.x = fminf(fmaxf(q.x, 0.f), qf);
          if (fabsf(q.x - rintf(q.x)) > 0.5f - 6.103515625e-05f) {
            const double k = fmin(fmax(rint(static_cast<double>(v[e]) / s) + z, 0.0), qmax);
            mq[e] = static_cast<uint32_t>(k);
          }
        }
      }
      uint32_t p[4];
#pragma unroll
      for (int w = 0; w < 4; ++w)
        p[w] = __byte_perm(__byte_perm(mq[4 * w], mq[4 * w + 1], 0x0040),
                           __byte_perm(mq[4 * w + 2], mq[4 * w + 3], 0x0040), 0x5410);
      *reinterpret_cast<uint4*>(crow + blk * 128 + li * 16) = make_uint4(p[0], p[1], p[2], p[3]);
    }
    __syncwarp();
  }
}

}  // namespace dtq_fq
