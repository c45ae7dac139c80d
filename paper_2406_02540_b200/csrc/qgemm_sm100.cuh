// qgemm_sm100.cuh -- W8A8 / W4A8 quantized linear on sm_100a tensor cores.
//
//   acc[t,o] = sum_c x_u8[t,c] * w_s8[o,c]                (tcgen05.mma kind::i8,
//                                                          u8 x s8 -> s32 in TMEM)
//   acc     -= z_x[t] * sum_c w_s8[o,c]                   (qgemm.cpp:60)
//   y[t,o]   = s_x[t] * s_w[o] * acc + bias[o]            (qgemm.cpp:61-63)
//
// Persistent, warp-specialised, one CTA (or CTA pair) per SM:
//   epilogue warps (8 for W8A8, 4 for W4A8; low warp ids): tcgen05.ld 32
//               TMEM lanes x 32 columns, zero-point correction + dequant
//               (packed fp32x2) + bias + cast, swizzled smem staging, TMA
//               bulk stores (or coalesced 128-bit stores for unaligned y)
//   converter warps (W4A8 only): packed [BN x 64 B] nibbles -> s8 in the
//               canonical SWIZZLE_128B K-major layout
//   TMA warp    producer: A tile 128 x 128 B and B tile BN x 128 B (or BN/2
//               rows per CTA of a pair) per k-block into a kStages ring
//   MMA warp    TMEM allocator + single-thread MMA issuer (4 x K=32 MMAs per
//               k-block); tcgen05.commit frees smem stages and publishes a
//               finished accumulator
// TMEM holds two BN-column s32 accumulators so the epilogue of tile i
// overlaps the main loop of tile i+1.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

#include "gelu.cuh"
#include "ptx.cuh"

namespace dtq_gemm {

enum OutKind : int {
  kOutF16 = 0,
  kOutBF16 = 1,
  kOutF32 = 2,
  kOutS32 = 3,
  kOutNone = 4  // diagnostics only: drain TMEM without an epilogue (main-loop speed)
};

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
  int tma_store;        // 1: y rows 16-byte aligned -> TMA bulk stores (tmY valid)
  unsigned long long* probe;  // diagnostics: per-CTA wait-cycle counters (or nullptr)
  int dbg;              // diagnostics: 0 full epilogue, 2 TMEM loads only,
                        // 3 loads + dequant math, 4 + smem staging (no stores)
  const uint8_t* w4;    // W4A8 single-CTA tiles: packed nibbles [N, ld4] (read by the
  int64_t ld4;          // converter warps straight from L2)
  // Row flags (forward with the tile quantizer running concurrently): per
  // 128-row block, the number of rows whose codes / s_x / z_x are stored.
  // nullptr: the codes are complete before the kernel starts (griddepcontrol
  // .wait).  With flags, tiles run n-fastest (early row blocks first), the
  // producer and the epilogue wait on their block, and the last CTA to exit
  // resets the counters (and the `done` ticket) to zero for the next forward.
  uint32_t* ready;
  uint32_t* done;
  int mblocks;          // ceil(M / 128): counters to reset
  int act;              // activation on y in the epilogue: 0 none, 1 GELU (fp outputs)
  int b_pre;            // 1: B is a layer constant (the handle's weights), loaded for the
                        // first stages before griddepcontrol.wait; 0: B is written by
                        // an earlier kernel of this forward (W4 weights unpacked to s8)
};

constexpr int BM = 128;
constexpr int BK = 128;  // bytes (= int8 elements) per k-block: one 128-byte swizzle atom
#ifndef DTQ_CONV_WARPS
#define DTQ_CONV_WARPS 8
#endif
constexpr int kConvWarps = DTQ_CONV_WARPS;
// single-CTA W4A8: the converter warps split into groups that take turns on
// k-blocks, so each group has kConvGroups k-blocks of MMA time per unpack
// (its barrier / proxy-fence latency overlaps the other group's work)
#ifndef DTQ_CONV_GROUPS
#define DTQ_CONV_GROUPS 2
#endif
constexpr int kConvGroups = DTQ_CONV_GROUPS;
// epilogue warps: 8 (two per TMEM lane quarter, each half of the columns);
// W4A8 adds 8 nibble-converter warps.  Measured at fc1 (16384 x 4608 x 1152):
// W8A8 with 4 / 8 / 16 epilogue warps 127 / 72 / 72 us; W4A8 with 4 / 8 / 16
// converters 164 / 140 / 226 us, and 8 epilogue warps on top 133 us.
#ifndef DTQ_W8_EPI_WARPS
#define DTQ_W8_EPI_WARPS 8
#endif
#ifndef DTQ_W4_EPI_WARPS
#define DTQ_W4_EPI_WARPS 8
#endif
template <bool kW4>
__host__ __device__ constexpr int epi_warps() {
  return kW4 ? DTQ_W4_EPI_WARPS : DTQ_W8_EPI_WARPS;
}

// W4A8 single-CTA tiles: the packed nibbles ride the TMA stage ring with A
// (1), or the converter warps load them from L2 with LDG (0)
#ifndef DTQ_W4_TMA_PACKED
#define DTQ_W4_TMA_PACKED 1
#endif
constexpr bool kW4TmaPacked = DTQ_W4_TMA_PACKED != 0;
// W4A8 single-CTA tiles at BN=128 run two 128-row M sub-tiles per CTA (M =
// 256, two TMEM accumulators per tile), so each unpacked B k-block feeds
// twice the MMA work
#ifndef DTQ_W4_M2
#define DTQ_W4_M2 1
#endif
template <int BN, bool kW4, bool k2Cta>
__host__ __device__ constexpr bool dual_m() {
  return DTQ_W4_M2 != 0 && kW4 && !k2Cta && BN == 128;
}
#ifndef DTQ_W4_CB
// W4A8: depth of the unpacked-B ring.  Two, so the stage ring (A + packed
// nibbles) can be four deep: measured 24.7 vs 26.3 us (3 + 3) and 32.1 us
// (2 + 4) at C3 fc1
#define DTQ_W4_CB 2
#endif
template <int BN, int kStages, bool kW4, bool k2Cta = false>
struct Smem {
  static constexpr bool kM2 = dual_m<BN, kW4, k2Cta>();
  static constexpr int kA = BM * BK * (kM2 ? 2 : 1);  // this CTA's A rows per stage
  static constexpr int kBRows = k2Cta ? BN / 2 : BN;   // a CTA pair splits B along N
  static constexpr int kB = kBRows * BK;               // s8 tile
  // (W4A8 converters load the packed nibbles from L2: no smem for them)
  // packed nibbles of this CTA's B rows per stage (single-CTA W4A8 on the
  // TMA path); CTA pairs' converters load them from L2
  static constexpr int kP = (kW4 && kW4TmaPacked) ? kBRows * (BK / 2) : 0;
  // staging buffers per epilogue warp (one when the budget is tight)
  // (W8A8 CTA pairs at BN=256 trade the second buffer for a sixth stage:
  // +1-2 % on the STDiT shapes)
  static constexpr int kEpiBufs =
      (epi_warps<kW4>() > 8 || (kP > 0 && (BN == 256 || kM2)) || (!kW4 && k2Cta && BN == 256))
          ? 1
          : 2;
  static constexpr int kEpi = epi_warps<kW4>() * kEpiBufs * 32 * 64;  // 32 rows x 64 B each
  static constexpr int kPar = 2 * 3 * BN * 4;             // {s_w, wsum, bias} x 2 tiles
  static constexpr int offA = 0;
  // W4A8: the unpacked s8 B tiles live in their own kCB-deep ring, decoupled
  // from the TMA ring (A + packed nibbles), so the TMA ring can be deep
  static constexpr int kCB = kW4 ? DTQ_W4_CB : kStages;
  static constexpr int offB = offA + kStages * kA;
  static constexpr int offP = offB + kCB * kB;
  static constexpr int offE = offP + kStages * kP;
  static constexpr int offPar = offE + kEpi;
  static constexpr int offBar = offPar + kPar;
  // full[kStages], empty[kStages], conv[kCB], bempty[kCB], tfull[2], tempty[2]
  static constexpr int kBars = kStages * 2 + kCB * 2 + 4;
  static constexpr int bytes = offBar + kBars * 8 + 16;
  static constexpr int alloc = bytes + 1024;  // manual 1024-byte alignment
  static_assert(alloc <= 227 * 1024, "shared memory budget exceeded");
};

template <int BN, bool kW4>
__host__ __device__ constexpr int num_threads() {
  return 32 * (2 + epi_warps<kW4>() + (kW4 ? kConvWarps : 0));
}

// One word of the handle's nibble layout (weight_pack_kernel in capi.cu:
// columns 8i..8i+7 as n = c ^ 8, the 4-bit two's complement of c - 8, byte
// k = n[k] | n[k+4] << 4) -> 8 bytes holding 16*(c - 8) as s8: a nibble in
// the HIGH half of a byte with a zero low half is exactly 16*(c - 8).
// Three instructions per 8 weights (the reference's stream order would need
// five: XOR, two masks, two byte permutes).  The GEMM folds the factor 16
// back out exactly (s_x/16 in the dequant, 16*sum(w) in the zero-point term,
// >>4 for the raw accumulator).
__device__ __forceinline__ uint2 w4_word_to_s8x8_x16(uint32_t w) {
  return make_uint2((w << 4) & 0xF0F0F0F0u, w & 0xF0F0F0F0u);
}

// k2Cta: a cluster of two CTAs on one TPC computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 issued by the leader (rank 0).  Each CTA loads its
// own 128 rows of A and half of the B rows; both TMA streams complete on the
// leader's `full` barrier, and the leader's MMA commits are multicast to the
// `empty` / `tfull` barriers of both CTAs.  Each CTA's TMEM holds its 128
// accumulator rows, drained by its own epilogue warps, which release the
// buffer on the leader's `tempty` barrier.
// Diagnostics modes (DTQ_DEBUG_GEMM_EPI) and the per-role wait probe
// (DTQ_DEBUG_GEMM_PROBE) exist only in builds with -DDTQ_GEMM_DIAG.
#ifdef DTQ_GEMM_DIAG
#define GEMM_DBG(g) ((g).dbg)
#define GEMM_PROBE(g) ((g).probe)
#else
#define GEMM_DBG(g) 0
#define GEMM_PROBE(g) static_cast<unsigned long long*>(nullptr)
#endif

#ifndef DTQ_CORES_MAXNREG
#define DTQ_CORES_MAXNREG 112
#endif
// kCoRes: the instance shares every SM with a tile-quantizer CTA (row flags):
// capped at 112 registers per thread so both CTAs' registers fit the SM (the
// others at 200, what 320 threads of one CTA per SM allow anyway).
// kAct: activation applied to the fp32 y before the cast (1 = GELU,
// toydit.cpp:83 -- the fc1 -> gelu of toydit.cpp:215-216 in fc1's epilogue)
template <int BN, int kStages, bool kW4, int kOut, bool k2Cta, bool kCoRes = false, int kAct = 0>
#ifdef DTQ_PLAIN_LB
__global__ void __launch_bounds__(num_threads<BN, kW4>(), 1)
#else
__global__ void __launch_bounds__(num_threads<BN, kW4>(), 1) __maxnreg__(kCoRes ? DTQ_CORES_MAXNREG : 200)
#endif
    qgemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmY, const GemmArgs g) {
  using namespace dtq_ptx;
  using L = Smem<BN, kStages, kW4, k2Cta>;
  constexpr bool kM2 = L::kM2;
  constexpr uint32_t kTmemCols = 2 * BN * (kM2 ? 2 : 1);
  constexpr int kTileM = (k2Cta || kM2) ? 2 * BM : BM;
  constexpr uint32_t kIdesc = idesc_i8_u8s8(k2Cta ? 2 * BM : BM, BN);

  constexpr int kEpiWarps = epi_warps<kW4>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for SWIZZLE_128B, kept as arithmetic on the shared
  // array so every access below compiles to LDS/STS (not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem + L::offA;
  uint8_t* sB = smem + L::offB;
  uint8_t* sP = smem + L::offP;
  uint8_t* sE = smem + L::offE;
  uint32_t* sPar = reinterpret_cast<uint32_t*>(smem + L::offPar);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::offBar);
  uint64_t* empty = full + kStages;
  uint64_t* conv = empty + kStages;   // [kCB] W4: unpacked B buffer ready
  uint64_t* bempty = conv + L::kCB;   // [kCB] W4: unpacked B buffer consumed
  uint64_t* tfull = bempty + L::kCB;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // Warp roles.  The SM's warp arbiter favours higher warp ids, so the
  // latency-critical single-thread roles (TMA producer, MMA issuer) take the
  // two highest ids and the epilogue / converter warps the low ones.
  constexpr uint32_t kTmaWarp = kEpiWarps + (kW4 ? kConvWarps : 0);
  constexpr uint32_t kMmaWarp = kTmaWarp + 1;
  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int total_tiles = g.tiles_m * g.tiles_n;
  const uint32_t rank = k2Cta ? cluster_ctarank() : 0;  // CTA rank in the pair
  // diagnostics: cycles spent in each role's waits (DTQ_DEBUG_GEMM_PROBE)
  unsigned long long pw0 = 0, pw1 = 0;
  auto timed_wait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc_cycles) {
    if (GEMM_PROBE(g) == nullptr) {
      mbar_wait(bar, par);
      return;
    }
    const long long t0 = clock64();
    mbar_wait(bar, par);
    acc_cycles += static_cast<unsigned long long>(clock64() - t0);
  };
  const int tile0 = k2Cta ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int tstride = k2Cta ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  // tile -> (m, n): m fastest (B tiles stay in L2 across a wave), or n fastest
  // with row flags (a wave needs only the first row blocks the quantizer
  // publishes)
  const bool flags = g.ready != nullptr;
  auto tile_m = [&](int t) { return flags ? t / g.tiles_n : t % g.tiles_m; };
  auto tile_n = [&](int t) { return flags ? t % g.tiles_n : t / g.tiles_m; };
  // rows of 128-row block `mb` to wait for (0 past M: TMA zero-fills them)
  auto block_rows = [&](int mb) { return g.M - mb * 128 < 128 ? g.M - mb * 128 : 128; };

  const long long t_start = clock64();
  const unsigned long long g_start_ns = GEMM_PROBE(g) ? globaltimer_ns() : 0ull;
  if (warp == kTmaWarp && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (g.tma_store) prefetch_tmap(&tmY);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int c = 0; c < L::kCB; ++c) {
      // one converter group per k-block; a CTA pair's leader counts both CTAs'
      mbar_init(&conv[c], (k2Cta ? 2 : 1) * (kConvWarps / kConvGroups));
      mbar_init(&bempty[c], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps * (k2Cta ? 2 : 1));
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (k2Cta)
      tmem_alloc_cta2<kTmemCols>(tmem_slot);
    else
      tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (k2Cta)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // The stage operations of the producer.  B (the weights, a layer constant)
  // may be loaded before griddepcontrol.wait; A (the codes) and the
  // per-token params come from the preceding quantizer kernel.
  auto arm = [&](int st) {
    if constexpr (k2Cta && kW4 && L::kP > 0) {
      // A of both CTAs lands on the leader's barrier; each CTA's packed
      // nibbles land on its OWN barrier, which its converters wait on
      mbar_arrive_expect_tx(&full[st], rank == 0 ? 2 * L::kA + L::kP : L::kP);
    } else if constexpr (k2Cta) {
      // both CTAs' bytes land on the leader's barrier; only it arms it
      // (W4A8 on the L2 path: A only, the converters fill B)
      if (rank == 0) mbar_arrive_expect_tx(&full[st], 2 * (L::kA + (kW4 ? 0 : L::kB)));
    } else {
      mbar_arrive_expect_tx(&full[st], L::kA + (kW4 ? L::kP : L::kB));  // kA: both sub-tiles with kM2
    }
  };
  auto load_b = [&](int st, int kb, int n0) {
    if constexpr (k2Cta && kW4 && L::kP > 0) {
      tma_load_2d(sP + st * L::kP, &tmB, &full[st], kb * (BK / 2), n0 + rank * L::kBRows);
    } else if constexpr (k2Cta) {
      if constexpr (!kW4)
        tma_load_2d_2sm(sB + st * L::kB, &tmB, mapa_shared(smem_u32(&full[st]), 0), kb * BK,
                        n0 + rank * L::kBRows);
    } else {
      if constexpr (!kW4)
        tma_load_2d(sB + st * L::kB, &tmB, &full[st], kb * BK, n0);
      else if constexpr (L::kP > 0)
        tma_load_2d(sP + st * L::kP, &tmB, &full[st], kb * (BK / 2), n0);
    }
  };
  auto load_a = [&](int st, int kb, int m0) {
    if constexpr (k2Cta) {
      tma_load_2d_2sm(sA + st * L::kA, &tmA, mapa_shared(smem_u32(&full[st]), 0), kb * BK, m0);
    } else {
      tma_load_2d(sA + st * L::kA, &tmA, &full[st], kb * BK, m0);
      if constexpr (kM2) tma_load_2d(sA + st * L::kA + BM * BK, &tmA, &full[st], kb * BK, m0 + BM);
    }
  };
  // B of the first stages before the wait: the weights' load latency
  // overlaps the quantizer's tail instead of following it
  int npre = 0;
  if (warp == kTmaWarp && lane == 0) {
    const int work = ((total_tiles - tile0 + tstride - 1) / tstride) * g.k_blocks;
    npre = !g.b_pre ? 0 : work < kStages ? work : kStages;
    int tile = tile0, kb = 0;
    for (int j = 0; j < npre; ++j) {
      arm(j);
      load_b(j, kb, tile_n(tile) * BN);
      if (++kb == g.k_blocks) {
        kb = 0;
        tile += tstride;
      }
    }
  }
  // A codes, s_x, z_x come from the preceding quantizer kernel: all of them
  // at once (griddepcontrol.wait), or row block by row block (flags)
  if (!flags) pdl_wait();
  pdl_launch_dependents();  // the next layer's quantizer may set up on freed SMs

  if (warp == kTmaWarp) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int j = 0;  // k-block sequence number (the first npre have their B already)
      for (int tile = tile0; tile < total_tiles; tile += tstride) {
        const int m0 = tile_m(tile) * kTileM + rank * BM;
        const int n0 = tile_n(tile) * BN;
        if (flags) {
          // this CTA's A rows (both sub-tiles with kM2) must be published
#pragma unroll
          for (int sub = 0; sub < (kM2 ? 2 : 1); ++sub) {
            const int mb = (m0 >> 7) + sub;
            if (mb * 128 < g.M) wait_rows_ready(g.ready + mb, static_cast<uint32_t>(block_rows(mb)));
          }
          fence_proxy_async_global();  // generic-proxy stores -> this thread's TMA reads
        }
        for (int kb = 0; kb < g.k_blocks; ++kb, ++j) {
          if (j >= npre) {
            timed_wait(&empty[s], ph ^ 1, pw0);
            arm(s);
            load_b(s, kb, n0);
          }
          load_a(s, kb, m0);
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      int cb = 0;            // W4: unpacked-B ring slot
      uint32_t cph = 0;
      for (int tile = tile0; tile < total_tiles; tile += tstride, ++it) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        timed_wait(&tempty[acc], aph ^ 1, pw1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN * (kM2 ? 2 : 1);
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          timed_wait(&full[s], ph, pw0);
          if constexpr (kW4) mbar_wait(&conv[cb], cph);
          tc_fence_after();
          const uint64_t bd = umma_desc_sw128(smem_u32(sB + (kW4 ? cb : s) * L::kB));
#pragma unroll
          for (int sub = 0; sub < (kM2 ? 2 : 1); ++sub) {  // kM2: both M sub-tiles, same B
            const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * L::kA + sub * BM * BK));
#pragma unroll
            for (int k = 0; k < BK / 32; ++k) {
              if constexpr (k2Cta)
                mma_i8_cta2(d, ad + 2 * k, bd + 2 * k, kIdesc, (kb | k) != 0 ? 1u : 0u);
              else
                mma_i8(d + sub * BN, ad + 2 * k, bd + 2 * k, kIdesc, (kb | k) != 0 ? 1u : 0u);
            }
          }
          if constexpr (k2Cta)
            mma_commit_cta2_mc(&empty[s], 0x3);
          else
            mma_commit(&empty[s]);
          if constexpr (kW4) {
            // the unpacked B buffer is free once these MMAs have read it
            if constexpr (k2Cta)
              mma_commit_cta2_mc(&bempty[cb], 0x3);
            else
              mma_commit(&bempty[cb]);
            if (++cb == L::kCB) {
              cb = 0;
              cph ^= 1;
            }
          }
          if (++s == kStages) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (k2Cta)
          mma_commit_cta2_mc(&tfull[acc], 0x3);
        else
          mma_commit(&tfull[acc]);
      }
    }
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // warp w owns TMEM lanes [32*(w%4), +32) = tile rows (lane = one row) and
    // one contiguous column range of the tile (BN / (kEpiWarps/4) columns).
    const uint32_t q = warp & 3;
    // (kM2: warps 0-3 drain M sub-tile 0, 4-7 sub-tile 1, all BN columns)
    constexpr int kColGroups = kM2 ? 1 : kEpiWarps / 4;
    constexpr int kCols = BN / kColGroups;
    const int cgrp = kM2 ? 0 : warp / 4;
    const int sub = kM2 ? static_cast<int>(warp >> 2) : 0;
    const int qrow = sub * BM + static_cast<int>(q) * 32;  // first tile row of this warp
    const int et = threadIdx.x;                        // index among epilogue threads
    constexpr int kBufs = L::kEpiBufs;
    uint8_t* stage = sE + warp * (kBufs * 32 * 64);  // 32 x 64 B staging buffer(s)
    constexpr int esize = (kOut == kOutF16 || kOut == kOutBF16 || kOut == kOutNone) ? 2 : 4;
    constexpr int kPieceCols = 64 / esize;             // columns per 64-byte staged row
    int buf = 0;
    int it = 0;
    const bool has_bias = g.bias != nullptr;
    // Per-column {s_w, -wsum, bias} and per-row {s_x, z_x} of the NEXT tile are
    // fetched into registers while the current tile is processed, then parked
    // in a double-buffered smem table: their global latency never stalls the
    // drain of TMEM.
    constexpr int kParPer = (BN + 32 * kEpiWarps - 1) / (32 * kEpiWarps);
    // The loads are unconditional (indices clamped into range) and their
    // values are used only when parked at the top of the next tile: any
    // select, negate or convert right after the load would make the warp
    // wait out the global latency before draining the current tile.
    uint32_t p_sw[kParPer], p_b[kParPer];
    int32_t p_ws[kParPer];
    uint32_t p_ok = 0;  // bit i: column i is inside the tile and N; bit 31: row < M
    double nsx = 0.0;
    int32_t nzx = 0;
    auto fetch = [&](int t) {
      const int tm0 = tile_m(t) * kTileM + rank * BM;
      const int tn0 = tile_n(t) * BN;
      p_ok = 0;
#pragma unroll
      for (int i = 0; i < kParPer; ++i) {
        const int col = tn0 + et + i * 32 * kEpiWarps;
        const bool okc = col < g.N && et + i * 32 * kEpiWarps < BN;
        const int cc = min(col, g.N - 1);
        p_ok |= okc ? (1u << i) : 0u;
        p_sw[i] = __float_as_uint(__ldg(g.s_w + cc));
        p_ws[i] = __ldg(g.wsum + cc);
        p_b[i] = has_bias ? __float_as_uint(__ldg(g.bias + cc)) : 0u;
      }
      const int row = tm0 + qrow + lane;
      p_ok |= row < g.M ? (1u << 31) : 0u;
      if (flags) {
        // s_x / z_x of rows the quantizer is still writing: wait for the
        // block, then read around L1 (no non-coherent __ldg)
        const int mb = (tm0 + qrow) >> 7;
        if (mb * 128 < g.M) wait_rows_ready(g.ready + mb, static_cast<uint32_t>(block_rows(mb)));
        nsx = __ldcg(g.s_x + min(row, g.M - 1));
        nzx = __ldcg(g.z_x + min(row, g.M - 1));
      } else {
        nsx = __ldg(g.s_x + min(row, g.M - 1));
        nzx = __ldg(g.z_x + min(row, g.M - 1));
      }
    };
    if (tile0 < total_tiles) fetch(tile0);
    for (int tile = tile0; tile < total_tiles; tile += tstride, ++it) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int m0 = tile_m(tile) * kTileM + rank * BM;
      const int n0 = tile_n(tile) * BN;
      uint32_t* par = sPar + acc * (3 * BN);
#pragma unroll
      for (int i = 0; i < kParPer; ++i) {
        const int c = et + i * 32 * kEpiWarps;
        if (c < BN) {
          const bool okc = (p_ok >> i) & 1u;
          par[c] = okc ? p_sw[i] : 0u;
          // W4: the unpacked weights are 16*w (w4_word_to_s8x8_x16), so is their sum
          par[BN + c] = okc ? static_cast<uint32_t>(-p_ws[i] * (kW4 ? 16 : 1)) : 0u;
          par[2 * BN + c] = okc ? p_b[i] : 0u;
        }
      }
      const bool rok = p_ok >> 31;
      const float sx = rok ? static_cast<float>(nsx) * (kW4 ? 0.0625f : 1.f) : 0.f;
      const int32_t zx = rok ? nzx : 0;
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      if (tile + tstride < total_tiles) fetch(tile + tstride);

      timed_wait(&tfull[acc], aph, pw0);
      tc_fence_after();
      // TMEM -> registers, 32 columns at a time; chunk cl+1 is in flight while
      // chunk cl is dequantised and stored (two register sets, full unroll)
      const uint32_t tbase =
          tmem_base + ((q * 32) << 16) + (acc * (kM2 ? 2 : 1) + sub) * BN + cgrp * kCols;
      // (CTAs of more than 448 threads -- 16 epilogue warps, or 8 epilogue +
      // 8 converter warps -- get one register set: the other warps hide the
      // load latency, and ~100 registers per thread remain)
      constexpr int kLdSets = num_threads<BN, kW4>() > 448 ? 1 : 2;
      uint32_t rr[kLdSets][32];
      tmem_ld_32x32b_x32(tbase, rr[0]);
      tmem_ld_wait_regs(rr[0]);
#pragma unroll
      for (int cl = 0; cl < kCols / 32; ++cl) {
        const int c = cgrp * (kCols / 32) + cl;  // 32-column chunk index within the tile
        uint32_t (&r)[32] = rr[cl % kLdSets];
        if (kLdSets == 1 && cl > 0) {
          tmem_ld_32x32b_x32(tbase + cl * 32, r);
          tmem_ld_wait_regs(r);
        }
        if (kLdSets == 2 && cl + 1 < kCols / 32)
          tmem_ld_32x32b_x32(tbase + (cl + 1) * 32, rr[(cl + 1) % kLdSets]);
        if (cl == kCols / 32 - 1) {
          // every TMEM read of this accumulator has completed: hand it back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if constexpr (k2Cta)
              mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));
            else
              mbar_arrive(&tempty[acc]);
          }
        }
        // diagnostics 14: the warps sharing the MMA warp's SMSP drain TMEM
        // only (their rows get no output); 13: they nap after each chunk
        if (GEMM_DBG(g) == 13 && (warp & 3) == (kMmaWarp & 3)) __nanosleep(300);
        if (kOut == kOutNone || GEMM_DBG(g) == 2 || (GEMM_DBG(g) >= 10 && GEMM_DBG(g) <= 12) ||
            (GEMM_DBG(g) == 14 && (warp & 3) == (kMmaWarp & 3))) {
          if (kLdSets == 2 && cl + 1 < kCols / 32) tmem_ld_wait_regs(rr[(cl + 1) % kLdSets]);
          // diagnostics 10-12: FFMA2 busy work the size of the dequant math
          // (~3.5 instructions per value) on all epilogue warps (10), only on
          // those sharing the MMA warp's SMSP (11), or only on the others (12)
          const int dg = GEMM_DBG(g);
          const bool same = (warp & 3) == (kMmaWarp & 3);
          if (dg == 10 || (dg == 11 && same) || (dg == 12 && !same)) {
            float2 a4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              a4[u] = make_float2(__uint_as_float(r[2 * u]), __uint_as_float(r[2 * u + 1]));
            const float2 m = make_float2(1.0001f, 0.9999f), c = make_float2(0.5f, -0.5f);
#pragma unroll 4
            for (int i = 0; i < 28; ++i)
#pragma unroll
              for (int u = 0; u < 4; ++u) a4[u] = __ffma2_rn(a4[u], m, c);
            if (a4[0].x + a4[1].y + a4[2].x + a4[3].y == 1.2345f) static_cast<uint32_t*>(g.y)[0] = 1u;
          }
          continue;
        }
#pragma unroll
        for (int piece = 0; piece < 32 / kPieceCols; ++piece) {
          // 16 output words = 64 bytes of this row
          uint32_t w[16];
#pragma unroll
          for (int j4 = 0; j4 < kPieceCols; j4 += 4) {
            const int cc = c * 32 + piece * kPieceCols + j4;
            const bool nolds = GEMM_DBG(g) == 7;  // diagnostics: params from registers, no LDS
            const uint4 sw4 = nolds ? make_uint4(0x3f800000u, 0x3f800000u, 0x3f800000u, 0x3f800000u)
                                    : *reinterpret_cast<const uint4*>(par + cc);
            const uint4 ws4 = nolds ? make_uint4(0u, 0u, 0u, 0u)
                                    : *reinterpret_cast<const uint4*>(par + BN + cc);
            // (no bias: skip the load -- the epilogue shares smem bandwidth with
            // the MMA operand reads and the TMA ring)
            const uint4 b4 = has_bias ? *reinterpret_cast<const uint4*>(par + 2 * BN + cc)
                                      : make_uint4(0u, 0u, 0u, 0u);
            const uint32_t swv[4] = {sw4.x, sw4.y, sw4.z, sw4.w};
            const uint32_t wsv[4] = {ws4.x, ws4.y, ws4.z, ws4.w};
            const uint32_t bv[4] = {b4.x, b4.y, b4.z, b4.w};
            float f[4];
            int32_t a32[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int j = piece * kPieceCols + j4 + u;
              a32[u] = static_cast<int32_t>(r[j]) + zx * static_cast<int32_t>(wsv[u]);  // -wsum
            }
            // dequant in packed fp32x2 (FMUL2 / FFMA2): y = acc * (s_x * s_w) + bias
#pragma unroll
            for (int u = 0; u < 4; u += 2) {
              const float2 sc = __fmul2_rn(make_float2(sx, sx),
                                           make_float2(__uint_as_float(swv[u]),
                                                       __uint_as_float(swv[u + 1])));
              const float2 yy = __ffma2_rn(
                  GEMM_DBG(g) == 15  // diagnostics: no I2FP (bits reinterpreted)
                      ? make_float2(__int_as_float(a32[u]), __int_as_float(a32[u + 1]))
                      : make_float2(static_cast<float>(a32[u]), static_cast<float>(a32[u + 1])),
                  sc,
                  make_float2(__uint_as_float(bv[u]), __uint_as_float(bv[u + 1])));
              if constexpr (kAct == 1) {
                const float2 gy = dtq_act::gelu2(yy);
                f[u] = gy.x;
                f[u + 1] = gy.y;
              } else {
                f[u] = yy.x;
                f[u + 1] = yy.y;
              }
            }
            if constexpr (kOut == kOutF16) {
              const __half2 h0 = __floats2half2_rn(f[0], f[1]);
              const __half2 h1 = __floats2half2_rn(f[2], f[3]);
              w[j4 / 2] = *reinterpret_cast<const uint32_t*>(&h0);
              w[j4 / 2 + 1] = *reinterpret_cast<const uint32_t*>(&h1);
            } else if constexpr (kOut == kOutBF16) {
              const __nv_bfloat162 h0 = __floats2bfloat162_rn(f[0], f[1]);
              const __nv_bfloat162 h1 = __floats2bfloat162_rn(f[2], f[3]);
              w[j4 / 2] = *reinterpret_cast<const uint32_t*>(&h0);
              w[j4 / 2 + 1] = *reinterpret_cast<const uint32_t*>(&h1);
            } else if constexpr (kOut == kOutF32) {
#pragma unroll
              for (int u = 0; u < 4; ++u) w[j4 + u] = __float_as_uint(f[u]);
            } else {
#pragma unroll
              for (int u = 0; u < 4; ++u) w[j4 + u] = static_cast<uint32_t>(a32[u] >> (kW4 ? 4 : 0));
            }
          }
          if (GEMM_DBG(g) == 3 || GEMM_DBG(g) == 7) {  // diagnostics: keep the math alive, skip staging + stores
            uint32_t x = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) x ^= w[i];
            if (x == 0x9E3779B9u && lane == 77) static_cast<uint32_t*>(g.y)[0] = x;
            continue;
          }
          if (GEMM_DBG(g) == 6) {  // diagnostics: direct 128-bit stores from registers, no staging
            const int col0d = n0 + c * 32 + piece * kPieceCols;
            const int rowd = m0 + qrow + lane;
            if (rowd < g.M) {
              uint8_t* dst = static_cast<uint8_t*>(g.y) +
                             (static_cast<int64_t>(rowd) * g.ldy + col0d) * esize;
#pragma unroll
              for (int gq = 0; gq < 4; ++gq)
                if (col0d + (gq + 1) * (16 / esize) <= g.N)
                  *reinterpret_cast<uint4*>(dst + 16 * gq) =
                      make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
            }
            continue;
          }
          // stage: row `lane`, 4 granules of 16 B, 64-byte swizzle (conflict-free)
          uint8_t* sb = stage + buf * (32 * 64);
          if (g.tma_store) {
            // the bulk store that last read this buffer must have finished reading it
            if (lane == 0) {
              const long long t0 = GEMM_PROBE(g) ? clock64() : 0;
              bulk_wait_read<kBufs - 1>();
              if (GEMM_PROBE(g)) pw1 += static_cast<unsigned long long>(clock64() - t0);
            }
            __syncwarp();
          }
#pragma unroll
          for (int gq = 0; gq < 4; ++gq)
            *reinterpret_cast<uint4*>(sb + lane * 64 + ((gq ^ ((lane >> 1) & 3)) * 16)) =
                make_uint4(w[4 * gq], w[4 * gq + 1], w[4 * gq + 2], w[4 * gq + 3]);
          const int col0 = n0 + c * 32 + piece * kPieceCols;
          if (GEMM_DBG(g) == 4) {  // diagnostics: staging written, no global stores
            __syncwarp();
            continue;
          }
          if (g.tma_store) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (GEMM_DBG(g) == 16)  // diagnostics: each CTA re-stores onto one tile of its own
                tma_store_2d(&tmY, sb, (col0 - n0) * esize,
                             static_cast<int>((blockIdx.x * BM) % static_cast<unsigned>(g.M)) + qrow);
              else
                tma_store_2d(&tmY, sb, col0 * esize, m0 + qrow);
              bulk_commit();
            }
            buf = (buf + 1) % kBufs;
          } else {
            __syncwarp();
            // coalesced copy-out: 4 lanes per row (64 contiguous bytes), 8 rows per step
#pragma unroll
            for (int st = 0; st < 4; ++st) {
              const int srow = st * 8 + (lane >> 2);
              const int gq = lane & 3;
              const int grow = m0 + qrow + srow;
              const int gcol = col0 + gq * (16 / esize);
              if (grow < g.M && gcol < g.N) {
                const uint4 v =
                    *reinterpret_cast<const uint4*>(sb + srow * 64 + ((gq ^ ((srow >> 1) & 3)) * 16));
                uint8_t* dst = static_cast<uint8_t*>(g.y) +
                               (static_cast<int64_t>(grow) * g.ldy + gcol) * esize;
                const int nel = min(16 / esize, g.N - gcol);
                if (nel == 16 / esize && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                  *reinterpret_cast<uint4*>(dst) = v;
                } else {
                  const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
                  for (int b = 0; b < nel * esize; ++b)
                    dst[b] = static_cast<uint8_t>(vv[b >> 2] >> (8 * (b & 3)));
                }
              }
            }
            __syncwarp();
          }
        }
        if (kLdSets == 2 && cl + 1 < kCols / 32) tmem_ld_wait_regs(rr[(cl + 1) % kLdSets]);
      }
    }
    if (g.tma_store && lane == 0) bulk_wait<0>();
  } else if constexpr (kW4 && L::kP > 0) {
    // ------------------------------------------------------------ nibble converters
    // TMA path: the packed nibbles of k-block kb land in the stage ring with
    // A (one TMA box of 64 B x this CTA's B rows, on this CTA's own barrier);
    // a converter group reads them from smem, unpacks and stores the s8 tile
    // for the MMA (a CTA pair's leader MMA reads both CTAs' halves).
    constexpr int kGW = kConvWarps / kConvGroups;              // warps per group
    const int cw = static_cast<int>(warp) - kEpiWarps;          // converter warp index
    const int grp = cw / kGW;
    const int ct = (cw % kGW) * 32 + static_cast<int>(lane);    // thread within the group
    constexpr int kIt = L::kBRows * 8 / (32 * kGW);
    const int total = ((total_tiles - tile0 + tstride - 1) / tstride) * g.k_blocks;
    for (int seq = grp; seq < total; seq += kConvGroups) {
      const int st = seq % kStages;
      const uint32_t sph = (seq / kStages) & 1;
      mbar_wait(&full[st], sph);  // A + packed nibbles of this k-block landed
      const uint8_t* src = sP + st * L::kP;
      uint2 v[kIt];
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int item = ct + i * 32 * kGW;
        v[i] = *reinterpret_cast<const uint2*>(src + (item >> 3) * 64 + (item & 7) * 8);
      }
      const int cb = seq % L::kCB;
      const uint32_t cph = (seq / L::kCB) & 1;
      mbar_wait(&bempty[cb], cph ^ 1);  // the MMA has finished with this B buffer
      uint8_t* dst = sB + cb * L::kB;
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int item = ct + i * 32 * kGW;
        const int r = item >> 3, j = item & 7;
        const uint2 o0 = w4_word_to_s8x8_x16(v[i].x), o1 = w4_word_to_s8x8_x16(v[i].y);
        *reinterpret_cast<uint4*>(dst + r * 128 + ((j ^ (r & 7)) * 16)) =
            make_uint4(o0.x, o0.y, o1.x, o1.y);
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        if constexpr (k2Cta)
          mbar_arrive_cluster_release(mapa_shared(smem_u32(&conv[cb]), 0));
        else
          mbar_arrive(&conv[cb]);
      }
    }
  } else if constexpr (kW4) {
    // ------------------------------------------------------------ nibble converters
    // The packed nibbles come straight from L2 (the whole packed B of a layer
    // is a few MB), one k-block ahead in registers, so shared memory carries
    // only the unpacked s8 tile.  8 consecutive threads read one row's 64
    // bytes.  In a CTA pair each CTA converts its own half of the B rows and
    // reports to the leader, whose MMA reads both halves.
    constexpr int kGW = kConvWarps / kConvGroups;              // warps per group
    const int cw = static_cast<int>(warp) - kEpiWarps;          // converter warp index
    const int grp = cw / kGW;
    const int ct = (cw % kGW) * 32 + static_cast<int>(lane);    // thread within the group
    constexpr int kIt = L::kBRows * 8 / (32 * kGW);
    auto load = [&](int t, int kb, uint2 (&v)[kIt]) {
      const int n0 = tile_n(t) * BN + rank * L::kBRows;
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int item = ct + i * 32 * kGW;
        const int r = item >> 3, j = item & 7;
        const int64_t row = min(n0 + r, g.N - 1);
        const int64_t off = static_cast<int64_t>(kb) * (BK / 2) + j * 8;
        v[i] = off < g.ld4 ? __ldg(reinterpret_cast<const uint2*>(g.w4 + row * g.ld4 + off))
                           : make_uint2(0u, 0u);
      }
    };
    // this group's k-blocks: sequence numbers grp, grp + kConvGroups, ...
    auto advance = [&](int& t, int& k) {
      for (int u = 0; u < kConvGroups; ++u)
        if (++k == g.k_blocks) {
          k = 0;
          t += tstride;
        }
    };
    int seq = grp;
    int tile = tile0, kb = 0;
    for (int u = 0; u < grp; ++u)
      if (++kb == g.k_blocks) {
        kb = 0;
        tile += tstride;
      }
    uint2 cur[kIt];
    if (tile < total_tiles) load(tile, kb, cur);
    while (tile < total_tiles) {
      int ntile = tile, nkb = kb;
      advance(ntile, nkb);
      uint2 nxt[kIt];
      // diagnostics (-DDTQ_GEMM_DIAG): 8 no loads / unpack / stores, 9 no
      // smem stores, 10 no proxy fence, 11 no loads
      const int cdbg = GEMM_DBG(g);
      if (ntile < total_tiles && cdbg != 8 && cdbg != 11) load(ntile, nkb, nxt);
      if (cdbg == 8 || cdbg == 11)
        for (int i = 0; i < kIt; ++i) nxt[i] = make_uint2(0x12345678u ^ i, 0u);
      const int cb = seq % L::kCB;
      const uint32_t cph = (seq / L::kCB) & 1;
      mbar_wait(&bempty[cb], cph ^ 1);  // the MMA has finished with this B buffer
      uint8_t* dst = sB + cb * L::kB;
#pragma unroll
      for (int i = 0; i < kIt; ++i) {
        const int item = ct + i * 32 * kGW;
        const int r = item >> 3, j = item & 7;
        const uint2 o0 = w4_word_to_s8x8_x16(cur[i].x), o1 = w4_word_to_s8x8_x16(cur[i].y);
        if (cdbg == 8 || cdbg == 9) {
          if ((o0.x ^ o1.y) == 0xFFFFFFFFu) dst[0] = 1;  // keep the math alive
          continue;
        }
        *reinterpret_cast<uint4*>(dst + r * 128 + ((j ^ (r & 7)) * 16)) =
            make_uint4(o0.x, o0.y, o1.x, o1.y);
      }
      if (cdbg != 10)
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the MMA (async proxy)
      __syncwarp();
      if (lane == 0) {
        if constexpr (k2Cta)
          mbar_arrive_cluster_release(mapa_shared(smem_u32(&conv[cb]), 0));
        else
          mbar_arrive(&conv[cb]);
      }
#pragma unroll
      for (int i = 0; i < kIt; ++i) cur[i] = nxt[i];
      tile = ntile;
      kb = nkb;
      seq += kConvGroups;
    }
  }

  if (GEMM_PROBE(g) != nullptr && lane == 0) {
    // [cta][slot]: 0 tma empty-wait, 1 mma full-wait, 2 mma tempty-wait,
    // 3 epi0 tfull-wait, 4 epi0 store-drain-wait, 5 total cycles (warp 0)
    unsigned long long* pr = GEMM_PROBE(g) + blockIdx.x * 8;
    if (warp == kTmaWarp) pr[0] = pw0;
    if (warp == kMmaWarp) { pr[1] = pw0; pr[2] = pw1; }
    if (warp == 0) {
      pr[3] = pw0;
      pr[4] = pw1;
      pr[5] = clock64() - t_start;
      pr[6] = g_start_ns;            // CTA start / end (globaltimer): timelines
      pr[7] = globaltimer_ns();
    }
  }
  tc_fence_before();
  if constexpr (k2Cta)
    cluster_sync();
  else
    __syncthreads();
  if (flags && threadIdx.x == 0) {
    // every row flag this CTA reads has been read: the last CTA out resets
    // them for the next forward (which can only start its quantizer after
    // this grid completes)
    __threadfence();
    if (atomicAdd(g.done, 1u) == gridDim.x - 1) {
      for (int i = 0; i < g.mblocks; ++i) g.ready[i] = 0u;
      *g.done = 0u;
      __threadfence();
    }
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (k2Cta)
      tmem_dealloc_cta2<kTmemCols>(tmem_base);
    else
      tmem_dealloc<kTmemCols>(tmem_base);
  }
}

#undef GEMM_DBG
#undef GEMM_PROBE

}  // namespace dtq_gemm
