// fused_quant_tile.cuh -- tile-pipelined fused quantizer (fp32 "fast" mode).
//
// Same contract as fq_fast_kernel (fused_quant_fast.cuh), with a
// decomposition built for instruction count and latency hiding:
//
//   TWO LANES (l and l+16 of a warp) OWN ONE 128-COLUMN BLOCK OF ONE ROW.
//
// Lane half p = lane / 16 holds the block elements e with bit 4 of e equal
// to p: four runs of 16 contiguous elements (e = 32m + 16p + 0..15), kept as
// 32 fp32 pairs P_k = (v_l, v_l+32) of local index l = 16m + (e & 15).  The
// 128-point Walsh-Hadamard transform then runs in the reference's stage
// order (balance.cpp:22-33): strides 1, 2, 4, 8 packed FADD2/FFMA2 in
// registers, stride 16 across the lane pair (shfl.xor 16), stride 32 packed,
// stride 64 inside each pair -- ~5 instructions per element.
//
// A CTA processes tiles of R rows x K columns (nb = K/128 blocks, pair q =
// 16*warp + lane%16 -> row q % R, block q / R; R <= 16), persistent over
// tiles, two CTAs per SM:
//   * the R input rows of a tile arrive by bulk async copies (cp.async.bulk,
//     one mbarrier per buffer) into a double buffer: tile i+1 is in flight
//     while tile i computes.  Row pitch = K*es + 16 bytes, so the 128-bit
//     reads of 8 rows per phase are bank-conflict free (R = 16);
//   * per-column multiplier (sign * 1/s_c * 1/sqrt(128), with the modulate
//     prologue's (1 + scale) and shift folded in) from a per-CTA smem table;
//   * row min / max: 3-input FMNMX3, pair shuffle, one smem exchange across
//     the nb blocks of a row = the ONLY barrier per tile; every thread then
//     derives its row's s, z in fp64 exactly as quant.cpp:90-124;
//   * codes: r = fma(v, 1/s, z + 1.5*2^23) rounds the exact product-sum once
//     (ties-even, low byte = code) -- one FFMA2 per two codes;
//   * kExactV (no prologue, smoothing or rotation: v is the exact input, so
//     the reference codes are reachable bit for bit): the exact residual
//     e = fma(v, 1/s, (z + 1.5*2^23) - r) is checked, and |e| > 1/2 - 2^-15
//     (|v/s - v*fl(1/s)| <= 2^-16 < the margin) re-checks that run of 16
//     values in registers and re-evaluates the flagged ones with an IEEE
//     fp64 divide (out of line; fp16 data has ~1e-4 exact ties);
//   * a lane pair's 2 x 16 codes per run are one contiguous 32-byte sector:
//     16-byte stores straight from registers, no staging, no barrier.
//
// Host contract: K % 128 == 0, K <= 8192, 16-byte aligned input rows and
// code rows, rotation block 128, blockDim = round_up(2*R*nb, 32), dynamic
// smem = fq_tile_layout(...).bytes.
#pragma once

#include <cstdlib>

#include "fused_quant.cuh"
#include "ptx.cuh"

namespace dtq_fq {

// Lanes per 128-column block: kQ = 4 for K <= 1152 (32 values per lane,
// <= 112 registers, two 288-thread CTAs per SM), kQ = 2 for wider rows and
// the LayerNorm prologue (64 values per lane, up to 576-thread CTAs).
// Derived per-lane shapes:
template <int kQ>
struct FqShape {
  static constexpr int kE = 128 / kQ;      // values per lane
  static constexpr int kPairs = kE / 2;    // fp32 pairs
  static constexpr int kRuns = kE / 16;    // 16-column runs
  static constexpr int kItems = 32 / kQ;   // (row, block) items per warp
};
// Four lanes per 128-column block (8-row tiles, 288-thread CTAs, two per
// SM) up to K = 1152; wider rows use two lanes per block in 576-thread CTAs.
// (Four lanes with shorter tiles for wider rows -- R = 4 / 2 / 1 -- measured
// slower: 109 vs 82 us at 16384 x 4608.)  DTQ_FQ_WIDE_K (diagnostics) moves
// the threshold.
constexpr int64_t kFqWideK = 1152;
__host__ inline int64_t fq_wide_k() {
  static const int64_t v = [] {
    const char* e = std::getenv("DTQ_FQ_WIDE_K");
    return e ? static_cast<int64_t>(std::atoll(e)) : kFqWideK;
  }();
  return v;
}
// The LayerNorm prologue takes the two-lane layout at every K: its extra
// statistics exchange per tile is amortised over 64 values per lane
// (measured 28.5 vs 30.4 us at 16384 x 1152).
__host__ inline int fq_lanes(int64_t K, int pro) {
  return (K <= fq_wide_k() && pro != kProLnModulate) ? 4 : 2;
}

constexpr int kFqMaxBuf = 4;  // input ring depth limit

struct TileLayout {
  size_t pitch_in;
  size_t off_in1, off_a, off_b, off_red, off_bar, bytes;
};

__host__ __device__ inline TileLayout fq_tile_layout(int64_t K, int R, int es, bool has_a,
                                                     bool has_b, int nbuf = 2) {
  TileLayout L;
  const size_t nb = static_cast<size_t>(K) / 128;
  L.pitch_in = static_cast<size_t>(K) * es + 16;
  L.off_in1 = static_cast<size_t>(R) * L.pitch_in;
  L.off_a = static_cast<size_t>(nbuf) * L.off_in1;  // nbuf-deep input ring
  L.off_b = L.off_a + (has_a ? static_cast<size_t>(K) * 4 : 0);
  L.off_red = L.off_b + (has_b ? static_cast<size_t>(K) * 4 : 0);
  // min/max pairs (double-buffered) + two LayerNorm partial arrays, nb x R each
  L.off_bar = L.off_red + nb * R * (2 * 8 + 4 + 4);
  L.off_bar = (L.off_bar + 7) / 8 * 8;
  L.bytes = L.off_bar + 8 * kFqMaxBuf;
  return L;
}

__host__ inline int fq_tile_threads(int64_t K, int R, int pro) {
  return static_cast<int>((fq_lanes(K, pro) * R * (K / 128) + 31) / 32 * 32);
}

// Per-column tables are stored pair-interleaved, (A[c], A[c + 64]) adjacent
// for c in the first half of each 128-column block, so a lane's multiplier
// pairs come straight out of 128-bit loads into aligned register pairs.
__device__ __forceinline__ int fq_pair_slot(int c) {
  const int j = c & 127;
  return (c & ~127) + (j < 64 ? 2 * j : 2 * (j - 64) + 1);
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float min3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

constexpr float kFqTie = 0.5f - 3.0517578125e-05f;  // 1/2 - 2^-15

// One exact code (quant.cpp:169-175 in fp64), out of line: called only for a
// value whose fp32 evaluation lies within 2^-15 of a rounding tie.
static __device__ __noinline__ uint32_t fq_exact_code(float x, double s, double z, double qmax) {
  return static_cast<uint32_t>(fmin(fmax(rint(static_cast<double>(x) / s) + z, 0.0), qmax));
}

// 16 raw elements at p (smem) -> fp32
template <typename Tin>
__device__ __forceinline__ void ld16(const uint8_t* p, float (&o)[16]) {
  float a[8], b[8];
  uint4 r0[Vec<Tin>::kWords], r1[Vec<Tin>::kWords];
#pragma unroll
  for (int w = 0; w < Vec<Tin>::kWords; ++w) {
    r0[w] = reinterpret_cast<const uint4*>(p)[w];
    r1[w] = reinterpret_cast<const uint4*>(p + 8 * sizeof(Tin))[w];
  }
  unpack<float>(r0, a, Tin());
  unpack<float>(r1, b, Tin());
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    o[i] = a[i];
    o[8 + i] = b[i];
  }
}

// value l (0..kE-1) of a lane: P[l % kPairs].x for l < kPairs, .y otherwise
#define FQ_V(P, l) ((l) < S::kPairs ? (P)[(l) % S::kPairs].x : (P)[(l) % S::kPairs].y)

// kE codes of one lane -> one 16-byte store per run (run m at dst + 16*kQ*m)
template <int kQ, bool kClamp, bool kExactV>
__device__ __forceinline__ void fq_tile_codes(const float2 (&P)[FqShape<kQ>::kPairs], float inv_sf,
                                              float zm, int qmax_i, double s_num, double s_den,
                                              double z, double qmax,
                                              uint8_t* __restrict__ dst) {
  const float2 inv2 = make_float2(inv_sf, inv_sf), zm2 = make_float2(zm, zm);
  const float2 neg = make_float2(-1.f, -1.f);
  const float lo = 12582912.0f, hi = 12582912.0f + static_cast<float>(qmax_i);
  using S = FqShape<kQ>;
  constexpr int kHalf = S::kRuns / 2;
  uint32_t w[4 * S::kRuns];  // run m (values 16m..16m+15) -> w[4m..4m+3]
  float em[S::kRuns];
#pragma unroll
  for (int m = 0; m < S::kRuns; ++m) em[m] = 0.f;
#pragma unroll
  for (int g = 0; g < 4; ++g) {  // pairs 4g..4g+3 of each 16-pair group
#pragma unroll
    for (int h = 0; h < kHalf; ++h) {
      uint32_t cx[4], cy[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 v = P[16 * h + 4 * g + u];
        float2 rr = __ffma2_rn(v, inv2, zm2);
        if constexpr (kExactV) {
          const float2 e = __ffma2_rn(v, inv2, __ffma2_rn(rr, neg, zm2));  // exact residual
          em[h] = fmaxf(em[h], fabsf(e.x));
          em[kHalf + h] = fmaxf(em[kHalf + h], fabsf(e.y));
        }
        if constexpr (kClamp) {
          rr.x = fminf(fmaxf(rr.x, lo), hi);
          rr.y = fminf(fmaxf(rr.y, lo), hi);
        }
        cx[u] = __float_as_uint(rr.x);
        cy[u] = __float_as_uint(rr.y);
      }
      // .x of pairs 16h + .. -> run h; .y -> run kHalf + h
      w[4 * h + g] = __byte_perm(__byte_perm(cx[0], cx[1], 0x0040),
                                 __byte_perm(cx[2], cx[3], 0x0040), 0x5410);
      w[4 * (kHalf + h) + g] = __byte_perm(__byte_perm(cy[0], cy[1], 0x0040),
                                           __byte_perm(cy[2], cy[3], 0x0040), 0x5410);
    }
  }
  if constexpr (kExactV) {
    unsigned runs = 0;
#pragma unroll
    for (int m = 0; m < S::kRuns; ++m) runs |= (em[m] > kFqTie ? 1u : 0u) << m;
    if (runs) {
      // possible fp32 ties: re-check each value of a flagged run in
      // registers; only a confirmed near-tie pays the out-of-line fp64 divide
      const double s = s_num / s_den;
#pragma unroll
      for (int m = 0; m < S::kRuns; ++m) {
        if (!((runs >> m) & 1u)) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x = FQ_V(P, 16 * m + i);
          const float rr = fmaf(x, inv_sf, zm);
          const float e = fmaf(x, inv_sf, zm - rr);
          if (fabsf(e) > kFqTie) {
            const uint32_t c = fq_exact_code(x, s, z, qmax);
            const uint32_t sh = 8u * (i & 3);
            w[4 * m + (i >> 2)] = (w[4 * m + (i >> 2)] & ~(0xffu << sh)) | (c << sh);
          }
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < S::kRuns; ++m)
    *reinterpret_cast<uint4*>(dst + 16 * kQ * m) =
        make_uint4(w[4 * m], w[4 * m + 1], w[4 * m + 2], w[4 * m + 3]);
}

// CTAs per SM the 288-thread kernels are register-capped for: two (112
// registers, 18 warps per SM).  Three (72 registers) spills in the LayerNorm
// and exact-code variants and measured slower everywhere at 16384 x 1152:
// no prologue 22.5 vs 23.3 us, modulate 24.4 vs 27.1, LayerNorm 33.1 vs
// 38.7, exact codes 20.7 vs 21.8.  DTQ_FQ_MINB (diagnostics build) sets it.
#ifndef DTQ_FQ_MINB
#define DTQ_FQ_MINB 2
#endif
// kWide: 576-thread CTAs (K > 1152, one per SM); otherwise <= 288 threads
// with registers capped for DTQ_FQ_MINB CTAs per SM
// Diagnostics modes (DTQ_DEBUG_FQ) exist only in builds with -DDTQ_FQ_DIAG:
// the extra paths cost registers in the product kernel.
#ifdef DTQ_FQ_DIAG
#define FQ_DBG(a) ((a).dbg)
#else
#define FQ_DBG(a) 0
#endif

// Rows [tile * R, +R) are stored: add them to their 128-row block's counter
// (release at gpu scope, after the CTA barrier that ordered every thread's
// stores).  The GEMM's producer waits for min(128, M - 128 b) rows.
__device__ __forceinline__ void fq_publish_rows(const FqArgs& a, int64_t tile, int R) {
  const int64_t row0 = tile * R;
  const int64_t n = a.M - row0 < R ? a.M - row0 : R;
  dtq_ptx::red_release_add(a.ready + (row0 >> 7), static_cast<uint32_t>(n));
}

template <typename Tin, bool kRot, bool kExactV, int kPro, bool kWide, int kR>
__global__ void __launch_bounds__(kWide ? 576 : 288, kWide ? 1 : DTQ_FQ_MINB)
    fq_tile_kernel(const FqArgs a) {
  // compile-time tile height and ring depth: the index arithmetic folds
  constexpr int R = kR;
  constexpr int nbuf = 2;
  constexpr int kFqQ = kWide ? 2 : 4;
  using S = FqShape<kFqQ>;
  constexpr int kFqE = S::kE, kFqPairs = S::kPairs, kFqRuns = S::kRuns, kFqItems = S::kItems;
  extern __shared__ __align__(128) uint8_t fq_smem[];
  constexpr int es = sizeof(Tin);
  constexpr bool has_b = kPro == kProModulate || kPro == kProLnModulate;
  const int K = static_cast<int>(a.K);
  const int nb = K >> 7;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const int p = lane / kFqItems;                         // lane's part of its block
  const int q = warp * kFqItems + (lane % kFqItems);    // (row, block) item index
  const int r = q & (R - 1);
  const int b_raw = q / R;
  const bool active = b_raw < nb;  // blockDim is rounded up to whole warps
  const int b = active ? b_raw : 0;
  const bool has_a = has_b || a.col_mul != nullptr;
  const TileLayout L = fq_tile_layout(K, R, es, has_a, has_b, nbuf);
  float* colA = reinterpret_cast<float*>(fq_smem + L.off_a);
  float* colB = reinterpret_cast<float*>(fq_smem + L.off_b);
  float2* red_mm = reinterpret_cast<float2*>(fq_smem + L.off_red);
  float* red_s1 = reinterpret_cast<float*>(fq_smem + L.off_red + static_cast<size_t>(nb) * R * 16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fq_smem + L.off_bar);  // [nbuf]
  const uint8_t* __restrict__ X = static_cast<const uint8_t*>(a.x);
  const uint32_t row_bytes = static_cast<uint32_t>(K) * es;

  const int64_t ntiles = (a.M + R - 1) / R;
  auto issue = [&](int64_t tile, int buf) {  // warp 0
    const int64_t row0 = tile * R;
    const int nval = static_cast<int>(a.M - row0 < R ? a.M - row0 : R);
    if (lane == 0) dtq_ptx::mbar_arrive_expect_tx(bar + buf, row_bytes * nval);
    __syncwarp();
    uint8_t* dst = fq_smem + buf * L.off_in1;
    if (lane < nval)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
          "[%3];" ::"r"(dtq_ptx::smem_u32(dst + lane * L.pitch_in)),
          "l"(reinterpret_cast<uint64_t>(X + ((row0 + lane) * a.ldx) * es)), "r"(row_bytes),
          "r"(dtq_ptx::smem_u32(bar + buf))
          : "memory");
  };
  int64_t tile = blockIdx.x;
#ifdef FQ_TILE_PROBE
  const unsigned long long pr_g0 = dtq_ptx::globaltimer_ns();
#endif
  // Without row flags the GEMM may launch at once: its prologue (TMEM, barriers,
  // descriptors) overlaps this kernel, and it waits for the whole grid.
  if (a.ready == nullptr) dtq_ptx::pdl_launch_dependents();
  // warp 0: barriers, then the first tile's copies (overlap the table setup).
  // Under programmatic dependent launch everything before pdl_wait() runs
  // while the kernel producing X drains: only layer constants are read there.
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < nbuf; ++i) dtq_ptx::mbar_init(bar + i, 1);
    dtq_ptx::fence_barrier_init();
  }
  // the folded table of a balanced layer is a layer constant: read it while
  // the producer of X drains.  A per-call table (dtq_quantize_rows derives it
  // stream-ordered right before this launch) is only visible after pdl_wait.
  const bool col_pre = !has_b && a.col_mul != nullptr && a.col_mul_const;
  if (col_pre) {
    for (int c0 = t; c0 < K; c0 += 8 * blockDim.x) {
      float m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * blockDim.x;
        m[u] = c < K ? __ldg(a.col_mul + c) : 1.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c < K) colA[fq_pair_slot(c)] = m[u];
      }
    }
  }
  dtq_ptx::pdl_wait();  // X (and the modulate vectors) come from earlier kernels
  // With row flags the GEMM may launch only now: it reads rows as they are
  // published, so it must never run while the kernel before this one (the
  // previous layer's GEMM) still does -- the row counters and the workspace
  // are then never shared between two forwards in flight.
  if (a.ready != nullptr) dtq_ptx::pdl_launch_dependents();
  if (warp == 0) {  // the ring's first nbuf - 1 tiles
    __syncwarp();
    for (int k = 0; k + 1 < nbuf; ++k)
      if (tile + k * static_cast<int64_t>(gridDim.x) < ntiles) issue(tile + k * gridDim.x, k);
  }
  // a W4A8 forward's s8 weights, expanded while the first tiles arrive (the
  // GEMM reads them after this grid completes)
  if (a.w4.src != nullptr)
    dtq_w4::unpack_range(a.w4, static_cast<int64_t>(blockIdx.x) * blockDim.x + t,
                         static_cast<int64_t>(gridDim.x) * blockDim.x);
  // folded per-column affine map with the per-call modulate vectors:
  // v -> v * A_c + B_c (or a per-call multiplier alone).  Loads are batched
  // 8 deep per thread.
  if (has_b || (a.col_mul != nullptr && !col_pre)) {
    for (int c0 = t; c0 < K; c0 += 8 * blockDim.x) {
      float m[8], sc[8], sh[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * blockDim.x;
        const bool in = c < K;
        m[u] = (in && a.col_mul != nullptr) ? __ldg(a.col_mul + c) : 1.f;
        if constexpr (has_b) {
          sc[u] = in ? __ldg(a.pro_scale + c) : 0.f;
          sh[u] = in ? __ldg(a.pro_shift + c) : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c < K) {
          if constexpr (has_b) {
            colA[fq_pair_slot(c)] = (1.f + sc[u]) * m[u];
            colB[fq_pair_slot(c)] = sh[u] * m[u];
          } else {
            colA[fq_pair_slot(c)] = m[u];
          }
        }
      }
    }
  }
  __syncthreads();
  const int qmax_i = (1 << a.bits) - 1;
  const double qmax = static_cast<double>(qmax_i);
  const float sg16 = (p & 1) ? -1.f : 1.f;
  const float sg32 = (p & 2) ? -1.f : 1.f;
  const int c0 = b * 128 + 16 * p;  // first column of run 0; run m at + 16*kFqQ*m

  // diagnostics (built with -DFQ_TILE_PROBE, DTQ_DEBUG_FQ_PROBE=1): per-CTA
  // cycles in data waits, in the tile barrier and in total (warp 1, lane 0)
#ifdef FQ_TILE_PROBE
  const bool probe = a.probe != nullptr && t == 32;
#else
  constexpr bool probe = false;
#endif
#ifdef FQ_TILE_PROBE
  long long pr_t0 = probe ? clock64() : 0;
#endif
  long long pr_wait = 0, pr_bar = 0;
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const int buf = it % nbuf;
    const int64_t row = tile * R + r;
    const bool ok = active && row < a.M;
    // prefetch nbuf - 1 tiles ahead into the buffer consumed last iteration
    // (every thread loaded it into registers before that iteration's barrier)
    {
      const int64_t ahead = tile + static_cast<int64_t>(nbuf - 1) * gridDim.x;
      if (warp == 0 && ahead < ntiles) {
        dtq_ptx::fence_proxy_async_smem();
        issue(ahead, (it + nbuf - 1) % nbuf);
      }
    }
    {
      const long long w0 = probe ? clock64() : 0;
      dtq_ptx::mbar_wait(bar + buf, (it / nbuf) & 1);
      if (probe) pr_wait += clock64() - w0;
    }

    // ---- 1. own kFqE values -> registers: run m = columns c0 + 16*kFqQ*m + 0..15;
    // runs m < kFqRuns/2 fill P[16m + i].x, the others .y
    float2 P[kFqPairs];
    {
      const uint8_t* src = fq_smem + buf * L.off_in1 + r * L.pitch_in + c0 * es;
#pragma unroll
      for (int m = 0; m < kFqRuns / 2; ++m) {
        float lo[16], hi[16];
        ld16<Tin>(src + 16 * kFqQ * m * es, lo);
        ld16<Tin>(src + (16 * kFqQ * m + 64) * es, hi);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          P[16 * m + i] = make_float2(lo[i], hi[i]);
          // GELU as the values arrive, 16 pairs at a time: fewer values live
          // beside its temporaries than in one pass over all of P (the
          // 576-thread wide variant is capped at 96 registers)
          if constexpr (kPro == kProGelu) P[16 * m + i] = gelu2(P[16 * m + i]);
        }
      }
    }

    if (FQ_DBG(a) == 3) {  // diagnostics: the memory pipeline alone (raw bits out, no math)
      if (ok) {
        uint8_t* dst = a.codes + row * a.ldc + c0;
#pragma unroll
        for (int m = 0; m < kFqRuns; ++m) {
          const float2* Q = P + 16 * (m % (kFqRuns / 2));
          *reinterpret_cast<uint4*>(dst + 16 * kFqQ * m) =
              make_uint4(__float_as_uint(Q[0].x) ^ __float_as_uint(Q[1].y),
                         __float_as_uint(Q[2].x) ^ __float_as_uint(Q[3].y),
                         __float_as_uint(Q[4].x) ^ __float_as_uint(Q[5].y),
                         __float_as_uint(Q[6].x) ^ __float_as_uint(Q[7].y));
        }
      }
      __syncthreads();
      continue;
    }
    // ---- 2. prologue
    if constexpr (kPro == kProLnModulate) {
      // LayerNorm statistics in ONE exchange: per-thread mean and M2 (two
      // passes over registers), merged across the lanes of a block and then
      // across the row's blocks with Chan et al.'s pairwise update (equal
      // counts), so a single CTA barrier suffices
      float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < kFqPairs; ++k) s2 = __fadd2_rn(s2, P[k]);
      float lm = (s2.x + s2.y) * (1.f / kFqE);
      float2 q2 = make_float2(0.f, 0.f);
      {
        const float2 nm = make_float2(-lm, -lm);
#pragma unroll
        for (int k = 0; k < kFqPairs; ++k) {
          const float2 d = __fadd2_rn(P[k], nm);
          q2 = __ffma2_rn(d, d, q2);
        }
      }
      float lM2 = q2.x + q2.y;
      float n = static_cast<float>(kFqE);
#pragma unroll
      for (int o = kFqItems; o < 32; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, lm, o);
        const float oM2 = __shfl_xor_sync(0xffffffffu, lM2, o);
        const float d = om - lm;
        lm = fmaf(d, 0.5f, lm);
        lM2 = lM2 + oM2 + d * d * (0.5f * n);
        n *= 2.f;
      }
      // rows shorter than a warp's items (R < kFqItems): fold the warp's
      // other blocks of the same row first (count-aware: items past the
      // last block carry no data), so the cross-warp merge reads one
      // partial per warp, not one per block
      float ln_n = 128.f;
      if (!active) {  // items past the last block: no data, no weight
        lm = 0.f;
        lM2 = 0.f;
        ln_n = 0.f;
      }
#pragma unroll
      for (int o = R; o < kFqItems; o <<= 1) {
        const float om = __shfl_xor_sync(0xffffffffu, lm, o);
        const float oM2 = __shfl_xor_sync(0xffffffffu, lM2, o);
        const float on = __shfl_xor_sync(0xffffffffu, ln_n, o);
        const float nn = ln_n + on;
        const float inv = nn > 0.f ? __frcp_rn(nn) : 0.f;
        const float d = om - lm;
        lm = fmaf(d, on * inv, lm);
        lM2 = lM2 + oM2 + d * d * (ln_n * on * inv);
        ln_n = nn;
      }
      float2* red_ln = reinterpret_cast<float2*>(red_s1);  // (mean, M2) per (warp, row)
      if (lane < R) red_ln[warp * R + r] = make_float2(lm, lM2);
      __syncthreads();
      // warp j holds blocks [j*kBpw, (j+1)*kBpw) of the row
      constexpr int kBpw = kFqItems / R;
      float2 st = red_ln[r];
      float st_n = 128.f * static_cast<float>(min(kBpw, nb));
      const int nw = (nb + kBpw - 1) / kBpw;
      for (int j = 1; j < nw; ++j) {
        const float2 o = red_ln[j * R + r];
        const float on = 128.f * static_cast<float>(min(kBpw, nb - j * kBpw));
        const float d = o.x - st.x;
        const float inv = __frcp_rn(st_n + on);
        st.x = fmaf(d, on * inv, st.x);
        st.y = st.y + o.y + d * d * (st_n * on * inv);
        st_n += on;
      }
      const float mean = st.x;
      const float rstd = rsqrtf(st.y / static_cast<float>(K) + a.eps);
      const float2 r2 = make_float2(rstd, rstd), o2 = make_float2(-mean * rstd, -mean * rstd);
#pragma unroll
      for (int k = 0; k < kFqPairs; ++k) P[k] = __ffma2_rn(P[k], r2, o2);
    }

    // ---- 3. folded column map, then the transform
    if (has_a && FQ_DBG(a) != 4) {
#pragma unroll
      for (int m = 0; m < kFqRuns / 2; ++m) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          // pairs 16m + 4g .. +3: .x columns jx = 16p + 16*kQ*m + 4g + (0..3) of
          // block b, .y columns jx + 64 -> pair slots b*64 + jx (interleaved)
          const int base = b * 64 + 16 * p + 16 * kFqQ * m + 4 * g;
          const float4 a01 = *reinterpret_cast<const float4*>(
              reinterpret_cast<const float2*>(colA) + base);
          const float4 a23 = *reinterpret_cast<const float4*>(
              reinterpret_cast<const float2*>(colA) + base + 2);
          float2* Q = P + 16 * m + 4 * g;
          if constexpr (has_b) {
            const float4 b01 = *reinterpret_cast<const float4*>(
                reinterpret_cast<const float2*>(colB) + base);
            const float4 b23 = *reinterpret_cast<const float4*>(
                reinterpret_cast<const float2*>(colB) + base + 2);
            Q[0] = __ffma2_rn(Q[0], make_float2(a01.x, a01.y), make_float2(b01.x, b01.y));
            Q[1] = __ffma2_rn(Q[1], make_float2(a01.z, a01.w), make_float2(b01.z, b01.w));
            Q[2] = __ffma2_rn(Q[2], make_float2(a23.x, a23.y), make_float2(b23.x, b23.y));
            Q[3] = __ffma2_rn(Q[3], make_float2(a23.z, a23.w), make_float2(b23.z, b23.w));
          } else {
            Q[0] = __fmul2_rn(Q[0], make_float2(a01.x, a01.y));
            Q[1] = __fmul2_rn(Q[1], make_float2(a01.z, a01.w));
            Q[2] = __fmul2_rn(Q[2], make_float2(a23.x, a23.y));
            Q[3] = __fmul2_rn(Q[3], make_float2(a23.z, a23.w));
          }
        }
      }
    }
    if (kRot && FQ_DBG(a) != 1 && FQ_DBG(a) != 4) {
      const float2 neg = make_float2(-1.f, -1.f);
      auto stage = [&](int h) {  // local stride h over the pair index
#pragma unroll
        for (int k = 0; k < kFqPairs; ++k)
          if ((k & h) == 0) {
            const float2 sm = __fadd2_rn(P[k], P[k + h]);
            const float2 df = __ffma2_rn(P[k + h], neg, P[k]);
            P[k] = sm;
            P[k + h] = df;
          }
      };
      stage(1);  // element stride 1
      stage(2);  // 2
      stage(4);  // 4
      stage(8);  // 8
      auto xlane = [&](int o, float sgn) {  // element stride 16 / 32 across lanes
        const float2 sg = make_float2(sgn, sgn);
#pragma unroll
        for (int k = 0; k < kFqPairs; ++k) {
          const float ox = __shfl_xor_sync(0xffffffffu, P[k].x, o);
          const float oy = __shfl_xor_sync(0xffffffffu, P[k].y, o);
          P[k] = __ffma2_rn(P[k], sg, make_float2(ox, oy));
        }
      };
      if (FQ_DBG(a) != 5) xlane(kFqItems, sg16);  // element stride 16
      if constexpr (kFqQ == 4) {
        if (FQ_DBG(a) != 5) xlane(2 * kFqItems, sg32);  // element stride 32
      }
      else
        stage(16);  // element stride 32 (local stride 16)
#pragma unroll
      for (int k = 0; k < kFqPairs; ++k)  // element stride 64: inside each pair, one
        // FFMA2 with both operands broadcast: (x + y, x - y) = y*(1, -1) + x
        P[k] = __ffma2_rn(make_float2(P[k].y, P[k].y), make_float2(1.f, -1.f),
                          make_float2(P[k].x, P[k].x));
    }
    if (a.status != nullptr && ok) {
      // non-finite input <=> non-finite sum (after the transform P[0].x of
      // lane half 0 IS the scaled block sum); re-checked element-wise
      float sum;
      if constexpr (kRot) {
        sum = P[0].x;
      } else {
        float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < kFqPairs; ++k) s2 = __fadd2_rn(s2, P[k]);
        sum = s2.x + s2.y;
      }
      if (!isfinite(sum)) {
        bool bad = false;
#pragma unroll
        for (int k = 0; k < kFqPairs; ++k) bad |= !isfinite(P[k].x) || !isfinite(P[k].y);
        if (bad) atomicOr(a.status, 1);
      }
    }

    // ---- 4. row min / max -> params (fp64, quant.cpp:90-124)
    {
      constexpr int kG = kFqPairs / 8;
      float mn4[4], mx4[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) mn4[i] = __int_as_float(0x7f800000), mx4[i] = -mn4[i];
#pragma unroll
      for (int i = 0; i < kG; ++i) {
        mn4[i] = fminf(P[8 * i].x, P[8 * i].y);
        mx4[i] = fmaxf(P[8 * i].x, P[8 * i].y);
#pragma unroll
        for (int k = 1; k < 8; ++k) {
          mn4[i] = min3f(mn4[i], P[8 * i + k].x, P[8 * i + k].y);
          mx4[i] = max3f(mx4[i], P[8 * i + k].x, P[8 * i + k].y);
        }
      }
      float mn = fminf(min3f(mn4[0], mn4[1], mn4[2]), mn4[3]);
      float mx = fmaxf(max3f(mx4[0], mx4[1], mx4[2]), mx4[3]);
#pragma unroll
      for (int o = kFqItems; o < 32; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      // R < kFqItems: the warp's other blocks of the same row (items past the
      // last block hold a copy of block 0 of their row: harmless here)
#pragma unroll
      for (int o = R; o < kFqItems; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane < R) red_mm[((it & 1) * nb + warp) * R + r] = make_float2(mn, mx);
    }
    {
      const long long b0 = probe ? clock64() : 0;
      __syncthreads();  // the one barrier per tile (also frees the input buffer)
      if (probe) pr_bar += clock64() - b0;
    }
    // every thread's code / param stores of the previous tile precede this
    // barrier: publish those rows to the GEMM waiting on their block
    if (a.ready != nullptr && t == 0 && it > 0) fq_publish_rows(a, tile - gridDim.x, R);
    // the row's min / max from the warps' partials: the 32 / R lanes of this
    // warp that share the row (lane & (R - 1) == r) each read every
    // (32 / R)-th partial, then a shuffle fold -- ceil(nwarp * R / 32) reads
    // per lane instead of nwarp (every lane, before the row-validity exit)
    float mn = __int_as_float(0x7f800000), mx = -mn;
    {
      const int nwarp = (nb * R + kFqItems - 1) / kFqItems;  // one partial per warp
      for (int j = lane / R; j < nwarp; j += 32 / R) {
        const float2 m = red_mm[((it & 1) * nb + j) * R + r];
        mn = fminf(mn, m.x);
        mx = fmaxf(mx, m.y);
      }
#pragma unroll
      for (int o = R; o < 32; o <<= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
    }
    if (!ok) continue;
    if (FQ_DBG(a) == 6) {  // diagnostics: codes with fixed parameters (no parameter math)
      fq_tile_codes<kFqQ, true, kExactV>(P, 0.01f + 1e-30f * mx, 128.f + 12582912.0f, qmax_i,
                                         1.0, 100.0, 128.0, qmax,
                                         a.codes + row * a.ldc + c0);
      continue;
    }
    // params (quant.cpp:90-124).  z needs rint(-lo / s) of the fp64 s: an
    // fp32 estimate is exact unless the quotient lies within 2^-10 of a
    // tie (then fp64); 1/s in fp32 suffices unless the codes must be exact
    // (kExactV).  The fp64 s itself is formed by the thread that stores it.
    const int qmax_i2 = qmax_i;
    bool clamp = a.symmetric || a.bits != 8;
    float zf, inv_sf;
    if (a.symmetric) {
      const float amax = fmaxf(fabsf(mn), fabsf(mx));
      zf = static_cast<float>(1 << (a.bits - 1));
      inv_sf = amax > 0.f ? static_cast<float>((1 << (a.bits - 1)) - 1) / amax : 1.f;
    } else if (mx == mn) {
      inv_sf = 1.f;
      zf = fminf(fmaxf(rintf(-mn), 0.f), static_cast<float>(qmax_i2));
      clamp = true;
    } else {
      const float lo = fminf(mn, 0.f), hi = fmaxf(mx, 0.f);
      inv_sf = static_cast<float>(qmax_i2) / (hi - lo);
      const float q = -lo * inv_sf;
      zf = fminf(fmaxf(rintf(q), 0.f), static_cast<float>(qmax_i2));
      if (fabsf(q - truncf(q) - 0.5f) < 1e-3f) {
        const double sd = (static_cast<double>(hi) - static_cast<double>(lo)) / qmax;
        zf = static_cast<float>(fmin(fmax(rint(-static_cast<double>(lo) / sd), 0.0), qmax));
      }
    }
    // s = num / den in fp64 (quant.cpp:90-124); only the writer lane forms
    // it (and the rare exact re-evaluation); kExactV needs fl32(1/s) = one
    // fp64 divide den / num per thread
    const bool writer = b == 0 && p == 0;
    double num = 1.0, den = 1.0;  // the fp64 s = num / den: writer and exact-code lanes only
    if (writer || kExactV) {
      const double dmn = static_cast<double>(mn), dmx = static_cast<double>(mx);
      if (a.symmetric) {
        const double amax = fmax(fabs(dmn), fabs(dmx));
        num = amax > 0.0 ? amax : 1.0;
        den = amax > 0.0 ? static_cast<double>((1 << (a.bits - 1)) - 1) : 1.0;
      } else if (dmx == dmn) {
        num = 1.0;
        den = 1.0;
      } else {
        num = fmax(dmx, 0.0) - fmin(dmn, 0.0);
        den = qmax;
      }
    }
    double s = 0.0;
    if (writer) {
      s = num / den;
      a.scale[row] = s;
      a.zero[row] = static_cast<int32_t>(zf);
    }
    if constexpr (kExactV) inv_sf = static_cast<float>(den / num);
    const double z = static_cast<double>(zf);
    const float zm = zf + 12582912.0f;

    // ---- 5. codes straight from registers
    uint8_t* dst = a.codes + row * a.ldc + c0;
    if (clamp)
      fq_tile_codes<kFqQ, true, kExactV>(P, inv_sf, zm, qmax_i, num, den, z, qmax, dst);
    else
      fq_tile_codes<kFqQ, false, kExactV>(P, inv_sf, zm, qmax_i, num, den, z, qmax, dst);
    // the GEMM reads these codes through TMA (async proxy)
    if (a.ready != nullptr) dtq_ptx::fence_proxy_async_global();
  }
  if (a.ready != nullptr) {  // publish the CTA's last tile
    __syncthreads();
    const int64_t nt = (a.M + R - 1) / R;
    if (t == 0 && blockIdx.x < nt) fq_publish_rows(a, tile - gridDim.x, R);
  }
#ifdef FQ_TILE_PROBE
  if (probe) {
    unsigned long long* pr = a.probe + blockIdx.x * 8;
    pr[0] = static_cast<unsigned long long>(pr_wait);
    pr[1] = static_cast<unsigned long long>(pr_bar);
    pr[2] = static_cast<unsigned long long>(clock64() - pr_t0);
    pr[3] = pr_g0;                        // CTA start (globaltimer ns)
    pr[4] = dtq_ptx::globaltimer_ns();    // CTA end
  }
#endif
}

#undef FQ_V
#undef FQ_DBG

}  // namespace dtq_fq
