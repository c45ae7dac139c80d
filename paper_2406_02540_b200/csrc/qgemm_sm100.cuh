// qgemm_sm100.cuh -- W8A8 / W4A8 quantized linear on sm_100a tensor cores.
//
//   acc[t,o] = sum_c x_u8[t,c] * w_s8[o,c]                (tcgen05.mma kind::i8,
//                                                          u8 x s8 -> s32 in TMEM)
//   acc     -= z_x[t] * sum_c w_s8[o,c]                   (qgemm.cpp:60)
//   y[t,o]   = s_x[t] * s_w[o] * acc + bias[o]            (qgemm.cpp:61-63)
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: A tile 128 x 128 B and B tile BN x 128 B per
//               k-block into a kStages ring (SWIZZLE_128B, mbarrier tx-count)
//   warp 1      TMEM allocator + single-thread MMA issuer (4 x K=32 MMAs per
//               k-block), tcgen05.commit frees smem stages and publishes a
//               finished accumulator
//   warps 2..5  epilogue: tcgen05.ld 32 lanes x 64 columns, zero-point
//               correction + dequant + bias + cast, swizzled smem staging,
//               coalesced 128-bit global stores
//   warps 6..9  (W4A8 only) nibble converters: packed [BN x 64 B] stage ->
//               s8 in the canonical SWIZZLE_128B K-major layout
// TMEM holds two BN-column s32 accumulators so the epilogue of tile i
// overlaps the main loop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "ptx.cuh"

namespace dtq_gemm {

enum OutKind : int { kOutF16 = 0, kOutBF16 = 1, kOutF32 = 2, kOutS32 = 3 };

struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n, k_blocks;
  const double* s_x;    // [M] per-token scale
  const int32_t* z_x;   // [M] per-token zero point
  const float* s_w;     // [N] per-channel weight scale
  const int32_t* wsum;  // [N] sum_c w_s8[o, c]
  const float* bias;    // [N] or nullptr
  void* y;
  int64_t ldy;          // elements
  int out_kind;
  int vec_store;        // 16-byte aligned rows -> 128-bit stores
};

constexpr int BM = 128;
constexpr int BK = 128;  // bytes (= int8 elements) per k-block: one 128-byte swizzle atom
constexpr int kEpiWarps = 4;
constexpr int kConvWarps = 4;

template <int BN, int kStages, bool kW4>
struct Smem {
  static constexpr int kA = BM * BK;                   // 16 KB
  static constexpr int kB = BN * BK;                   // s8 tile
  static constexpr int kP = kW4 ? BN * (BK / 2) : 0;   // packed nibbles
  static constexpr int kEpi = kEpiWarps * 32 * 128;    // 16 KB
  static constexpr int offA = 0;
  static constexpr int offB = offA + kStages * kA;
  static constexpr int offP = offB + kStages * kB;
  static constexpr int offE = offP + kStages * kP;
  static constexpr int offBar = offE + kEpi;
  static constexpr int kBars = kStages * 3 + 4;
  static constexpr int bytes = offBar + kBars * 8 + 16;
  static constexpr int alloc = bytes + 1024;  // manual 1024-byte alignment
};

template <int BN, bool kW4>
constexpr int num_threads() {
  return 32 * (2 + kEpiWarps + (kW4 ? kConvWarps : 0));
}

__device__ __forceinline__ uint32_t s4x8_to_s8x8_lo(uint32_t w) {
  // 8 LSB-first nibbles (codes, z = 8) -> bytes of (code - 8) for elements 0..3
  const uint32_t lo = w & 0x0F0F0F0Fu;         // elements 0, 2, 4, 6
  const uint32_t hi = (w >> 4) & 0x0F0F0F0Fu;  // elements 1, 3, 5, 7
  uint32_t e = __byte_perm(lo, hi, 0x5140);    // e0 e1 e2 e3
  e ^= 0x08080808u;                            // code - 8 as 4-bit two's complement
  return e | ((e & 0x08080808u) * 0x1Eu);      // sign-extend to 8 bits
}
__device__ __forceinline__ uint32_t s4x8_to_s8x8_hi(uint32_t w) {
  const uint32_t lo = w & 0x0F0F0F0Fu;
  const uint32_t hi = (w >> 4) & 0x0F0F0F0Fu;
  uint32_t e = __byte_perm(lo, hi, 0x7362);    // e4 e5 e6 e7
  e ^= 0x08080808u;
  return e | ((e & 0x08080808u) * 0x1Eu);
}

template <int BN, int kStages, bool kW4, int kOut>
__global__ void __launch_bounds__(num_threads<BN, kW4>(), 1)
    qgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const GemmArgs g) {
  using namespace dtq_ptx;
  using L = Smem<BN, kStages, kW4>;
  constexpr uint32_t kTmemCols = 2 * BN;
  constexpr uint32_t kIdesc = idesc_i8_u8s8(BM, BN);

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem + L::offA;
  uint8_t* sB = smem + L::offB;
  uint8_t* sP = smem + L::offP;
  uint8_t* sE = smem + L::offE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::offBar);
  uint64_t* empty = full + kStages;
  uint64_t* conv = empty + kStages;
  uint64_t* tfull = conv + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int total_tiles = g.tiles_m * g.tiles_n;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], kConvWarps);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
        const int m0 = (tile % g.tiles_m) * BM;
        const int n0 = (tile / g.tiles_m) * BN;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], L::kA + (kW4 ? L::kP : L::kB));
          tma_load_2d(sA + s * L::kA, &tmA, &full[s], kb * BK, m0);
          if constexpr (kW4)
            tma_load_2d(sP + s * L::kP, &tmB, &full[s], kb * (BK / 2), n0);
          else
            tma_load_2d(sB + s * L::kB, &tmB, &full[s], kb * BK, n0);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          mbar_wait(&full[s], ph);
          if constexpr (kW4) mbar_wait(&conv[s], ph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * L::kA));
          const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * L::kB));
#pragma unroll
          for (int k = 0; k < BK / 32; ++k)
            mma_i8(d, ad + 2 * k, bd + 2 * k, kIdesc, (kb | k) != 0 ? 1u : 0u);
          mma_commit(&empty[s]);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else if (warp < 2 + kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* stage = sE + (warp - 2) * (32 * 128);
    constexpr int esize = (kOut == kOutF16 || kOut == kOutBF16) ? 2 : 4;
    constexpr int cols_per_pass = 128 / esize;  // 64 (16-bit out) or 32 (32-bit out)
    int it = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int m0 = (tile % g.tiles_m) * BM;
      const int n0 = (tile / g.tiles_m) * BN;
      const int row = m0 + q * 32 + lane;
      const bool row_ok = row < g.M;
      const float sx = row_ok ? static_cast<float>(g.s_x[row]) : 0.f;
      const int32_t zx = row_ok ? g.z_x[row] : 0;

      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c) {
        uint32_t r[64];
        tmem_ld_32x32b_x64(tmem_base + ((q * 32) << 16) + acc * BN + c * 64, r);
        tmem_ld_wait();
        if (c == BN / 64 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        // column parameters: lane l holds columns l and l + 32 of this chunk
        const int cb = n0 + c * 64;
        float swv[2], bv[2];
        int32_t wsv[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = cb + h * 32 + lane;
          const bool ok = col < g.N;
          swv[h] = ok ? __ldg(g.s_w + col) : 0.f;
          wsv[h] = ok ? __ldg(g.wsum + col) : 0;
          bv[h] = (ok && g.bias) ? __ldg(g.bias + col) : 0.f;
        }
#pragma unroll
        for (int p = 0; p < 64 / cols_per_pass; ++p) {
          // stage row `lane`: cols_per_pass outputs = 128 bytes, 8 swizzled granules
#pragma unroll
          for (int gq = 0; gq < 8; ++gq) {
            uint32_t packed[4];
            if constexpr (esize == 2) {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float f2[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                  const int j = gq * 8 + e * 2 + u;  // column within the 64-chunk
                  const int h = j >> 5, src = j & 31;
                  const float sw = __shfl_sync(0xffffffffu, swv[h], src);
                  const int32_t ws = __shfl_sync(0xffffffffu, wsv[h], src);
                  const float b = __shfl_sync(0xffffffffu, bv[h], src);
                  const int32_t a32 = static_cast<int32_t>(r[j]) - zx * ws;
                  f2[u] = fmaf(static_cast<float>(a32), sx * sw, b);
                }
                if constexpr (kOut == kOutF16) {
                  const __half2 hv = __floats2half2_rn(f2[0], f2[1]);
                  packed[e] = *reinterpret_cast<const uint32_t*>(&hv);
                } else {
                  const __nv_bfloat162 hv = __floats2bfloat162_rn(f2[0], f2[1]);
                  packed[e] = *reinterpret_cast<const uint32_t*>(&hv);
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int j = p * 32 + gq * 4 + e;
                const int h = j >> 5, src = j & 31;
                const float sw = __shfl_sync(0xffffffffu, swv[h], src);
                const int32_t ws = __shfl_sync(0xffffffffu, wsv[h], src);
                const float b = __shfl_sync(0xffffffffu, bv[h], src);
                const int32_t a32 = static_cast<int32_t>(r[j]) - zx * ws;
                if constexpr (kOut == kOutS32)
                  packed[e] = static_cast<uint32_t>(a32);
                else
                  packed[e] = __float_as_uint(fmaf(static_cast<float>(a32), sx * sw, b));
              }
            }
            *reinterpret_cast<uint4*>(stage + lane * 128 + ((gq ^ (lane & 7)) * 16)) =
                make_uint4(packed[0], packed[1], packed[2], packed[3]);
          }
          __syncwarp();
          // coalesced write-out: 8 lanes per row (128 contiguous bytes), 4 rows per step
          const int col0 = cb + p * cols_per_pass;
#pragma unroll
          for (int st = 0; st < 8; ++st) {
            const int rr = st * 4 + (lane >> 3);
            const int gq = lane & 7;
            const int grow = m0 + q * 32 + rr;
            const int gcol = col0 + gq * (16 / esize);
            if (grow < g.M && gcol < g.N) {
              const uint4 v = *reinterpret_cast<const uint4*>(stage + rr * 128 + ((gq ^ (rr & 7)) * 16));
              uint8_t* dst = static_cast<uint8_t*>(g.y) + (static_cast<int64_t>(grow) * g.ldy + gcol) * esize;
              if (g.vec_store && gcol + 16 / esize <= g.N) {
                *reinterpret_cast<uint4*>(dst) = v;
              } else {
                const uint8_t* src = reinterpret_cast<const uint8_t*>(&v);
                const int nel = min(16 / esize, g.N - gcol);
                for (int b = 0; b < nel * esize; ++b) dst[b] = src[b];
              }
            }
          }
          __syncwarp();
        }
      }
    }
  } else if constexpr (kW4) {
    // ------------------------------------------------------------ nibble converters
    const int ct = threadIdx.x - 32 * (2 + kEpiWarps);  // 0..127
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
      for (int kb = 0; kb < g.k_blocks; ++kb) {
        mbar_wait(&full[s], ph);
        const uint8_t* src = sP + s * L::kP;
        uint8_t* dst = sB + s * L::kB;
        // BN rows x 8 granules of 16 output bytes (= 8 packed bytes each)
#pragma unroll 4
        for (int item = ct; item < BN * 8; item += 32 * kConvWarps) {
          const int r = item >> 3, j = item & 7;
          const uint2 w = *reinterpret_cast<const uint2*>(src + r * 64 + j * 8);
          const uint4 o = make_uint4(s4x8_to_s8x8_lo(w.x), s4x8_to_s8x8_hi(w.x),
                                     s4x8_to_s8x8_lo(w.y), s4x8_to_s8x8_hi(w.y));
          *reinterpret_cast<uint4*>(dst + r * 128 + ((j ^ (r & 7)) * 16)) = o;
        }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[s]);
        if (++s == kStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace dtq_gemm
