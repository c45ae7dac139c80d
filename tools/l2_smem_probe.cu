// l2_smem_probe.cu -- what bounds the GEMM main loop (diagnostics): the dense
// INT8 MMA stream of int8_ceiling.cu, with a second warp streaming bulk
// copies L2 -> shared memory at the same time (the GEMM producer's traffic,
// without the data dependency).  Reports the MMA rate and the copy bandwidth
// alone and together.  If the MMA rate holds while the copies run at the
// GEMM's required rate, the main loop is bound by L2 delivery; if it drops,
// by shared-memory bandwidth.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../paper_2406_02540_b200/csrc l2_smem_probe.cu -o _bin/l2_smem_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "ptx.cuh"

using namespace dtq_ptx;

constexpr int kChunk = 32 * 1024;  // one GEMM k-block of A + B per SM (pair tile)
constexpr int kRing = 3;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// mode bit 0: MMAs, bit 1: copies
__global__ void __launch_bounds__(128, 1) probe(int mode, int iters, int copies,
                                                const uint8_t* __restrict__ gsrc, int64_t span,
                                                unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                 // 16 KB A, 32 KB B (BN=256)
  uint8_t* sB = smem + 16384;
  uint8_t* ring = smem + 49152;       // kRing x 32 KB copy ring
  uint64_t* bar = reinterpret_cast<uint64_t*>(ring + kRing * kChunk);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + kRing + 1);
  for (int i = threadIdx.x; i < 49152 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, 7, 3, 1);
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    for (int i = 0; i <= kRing; ++i) mbar_init(bar + i, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const long long t0 = clock64();
  if ((mode & 1) && threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_i8_u8s8(128, 256);
    const uint64_t ad = umma_desc_sw128(smem_u32(sA)), bd = umma_desc_sw128(smem_u32(sB));
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8(tmem + (it & 1) * 256, ad + 2 * k, bd + 2 * k, idesc, k != 0 ? 1u : 0u);
    mma_commit(bar + kRing);
    mbar_wait(bar + kRing, 0);
  }
  if ((mode & 2) && threadIdx.x == 32) {
    // stream `copies` 32 KB chunks from a span of L2-resident memory
    const int64_t nchunks = span / kChunk;
    int64_t c = blockIdx.x * 7;
    for (int i = 0; i < copies; ++i) {
      const int s = i % kRing;
      if (i >= kRing) mbar_wait(bar + s, ((i / kRing) - 1) & 1);
      mbar_arrive_expect_tx(bar + s, kChunk);
      bulk_g2s(ring + s * kChunk, gsrc + (c % nchunks) * kChunk, kChunk, bar + s);
      c += 148;
    }
    for (int i = (copies > kRing ? copies - kRing : 0); i < copies; ++i)
      mbar_wait(bar + (i % kRing), (i / kRing) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// The GEMM's own pipeline shape with bulk copies instead of TMA tensor
// loads: a ring of `stages` x (16 KB A + 32 KB B); the MMA thread waits for a
// stage to land, issues its 4 MMAs (128 x 256 x 32) from it and commits the
// stage back; the producer thread refills a stage once its MMAs completed.
__global__ void __launch_bounds__(128, 1) pipeline(int stages, int kblocks,
                                                   const uint8_t* __restrict__ gsrc, int64_t span) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kStage = 49152;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int64_t nchunks = span / kStage;
  if (threadIdx.x == 32) {  // producer
    int64_t c = blockIdx.x * 5;
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(empty + s, ((kb / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(full + s, kStage);
      const uint8_t* src = gsrc + (c % nchunks) * kStage;
      bulk_g2s(smem + s * kStage, src, 16384, full + s);
      bulk_g2s(smem + s * kStage + 16384, src + 16384, 32768, full + s);
      c += 148;
    }
  } else if (threadIdx.x == 0) {  // MMA issuer
    constexpr uint32_t idesc = idesc_i8_u8s8(128, 256);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(full + s, (kb / stages) & 1);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(smem + s * kStage));
      const uint64_t bd = umma_desc_sw128(smem_u32(smem + s * kStage + 16384));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8(tmem + ((kb / 9) & 1) * 256, ad + 2 * k, bd + 2 * k, idesc, (kb % 9 | k) != 0 ? 1u : 0u);
      mma_commit(empty + s);
    }
    mma_commit(done);
    mbar_wait(done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// The same pipeline with the GEMM's own loads: TMA 2D boxes (128 rows x
// 128 B, SWIZZLE_128B) from a row-major [rows, 1152] u8 tensor (A: one box,
// B: two boxes of 128 rows) -- 128-byte row segments at a 1152-byte pitch.
__global__ void __launch_bounds__(128, 1) pipeline_tma(int stages, int kblocks, int rows,
                                                       const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kStage = 49152;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  if (threadIdx.x == 0) {
    prefetch_tmap(&tm);
    for (int i = 0; i < stages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 32) {  // producer
    int m = (blockIdx.x * 384) % (rows - 384);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(empty + s, ((kb / stages) & 1) ^ 1);
      mbar_arrive_expect_tx(full + s, kStage);
      const int k = (kb % 9) * 128;
      tma_load_2d(smem + s * kStage, &tm, full + s, k, m);
      tma_load_2d(smem + s * kStage + 16384, &tm, full + s, k, m + 128);
      tma_load_2d(smem + s * kStage + 32768, &tm, full + s, k, m + 256);
      if (kb % 9 == 8) m = (m + 148 * 384) % (rows - 384);
    }
  } else if (threadIdx.x == 0) {  // MMA issuer
    constexpr uint32_t idesc = idesc_i8_u8s8(128, 256);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(full + s, (kb / stages) & 1);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(smem + s * kStage));
      const uint64_t bd = umma_desc_sw128(smem_u32(smem + s * kStage + 16384));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8(tmem + ((kb / 9) & 1) * 256, ad + 2 * k, bd + 2 * k, idesc, (kb % 9 | k) != 0 ? 1u : 0u);
      mma_commit(empty + s);
    }
    mma_commit(done);
    mbar_wait(done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// The CTA-pair pipeline of the product GEMM (cta_group::2, 256 x 256 tiles):
// per k-block each CTA TMA-loads its 128 A rows and its 128 of the 256 B rows
// (16 + 16 KB) completing on the LEADER's full barrier; the leader issues
// 4 x tcgen05.mma.cta_group::2 and multicasts the commit to both CTAs' empty
// barriers, on which each CTA's producer waits before refilling.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    pipeline_pair(int stages, int kblocks, int rows, const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kStage = 32768;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * kStage);
  uint64_t* empty = full + stages;
  uint64_t* done = empty + stages;
  uint32_t* slot = reinterpret_cast<uint32_t*>(done + 1);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    prefetch_tmap(&tm);
    for (int i = 0; i < stages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc_cta2<512>(slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 32) {  // producer (both CTAs)
    int m = ((blockIdx.x >> 1) * 512) % (rows - 512);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(empty + s, ((kb / stages) & 1) ^ 1);
      const uint32_t lead_full = mapa_shared(smem_u32(full + s), 0);
      if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * kStage);
      const int k = (kb % 9) * 128;
      tma_load_2d_2sm(smem + s * kStage, &tm, lead_full, k, m + rank * 128);
      tma_load_2d_2sm(smem + s * kStage + 16384, &tm, lead_full, k, m + 256 + rank * 128);
      if (kb % 9 == 8) m = (m + 74 * 512) % (rows - 512);
    }
  } else if (threadIdx.x == 0 && rank == 0) {  // leader MMA issuer
    constexpr uint32_t idesc = idesc_i8_u8s8(256, 256);
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % stages;
      mbar_wait(full + s, (kb / stages) & 1);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(smem + s * kStage));
      const uint64_t bd = umma_desc_sw128(smem_u32(smem + s * kStage + 16384));
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8_cta2(tmem + ((kb / 9) & 1) * 256, ad + 2 * k, bd + 2 * k, idesc,
                    (kb % 9 | k) != 0 ? 1u : 0u);
      mma_commit_cta2_mc(empty + s, 0x3);
    }
    mma_commit_cta2_mc(done, 0x3);
  }
  if (threadIdx.x == 0) mbar_wait(done, 0);
  tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc_cta2<512>(tmem);
  }
}

int main() {
  const int sms = 148;
  const int64_t span = 10 << 20;  // 10 MB: the C2 GEMM's A + B footprint, L2-resident
  uint8_t* g;
  cudaMalloc(&g, span);
  cudaMemset(g, 1, span);
  unsigned long long* out;
  cudaMalloc(&out, sms * 8);
  const int smem = 49152 + kRing * kChunk + 64 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // per k-block (4 MMAs of 128x256x32 = 8.4 MOP per SM) the GEMM needs 32 KB
  // of A + B per SM (pair tiles): iters k-blocks <-> iters copies
  const int iters = 4000;
  const char* names[4] = {"", "mma only", "copies only", "mma + copies"};
  for (int mode = 1; mode <= 3; ++mode) {
    probe<<<sms, 128, smem>>>(mode, iters / 10, iters / 10, g, span, out);  // warm
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    probe<<<sms, 128, smem>>>(mode, iters, iters, g, span, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 2.0 * 128 * 256 * 128 * (double)iters * sms;
    const double bytes = (double)kChunk * iters * sms;
    printf("{\"mode\": \"%s\", \"ms\": %.3f, \"mma_tops\": %.0f, \"copy_tbs\": %.2f, \"err\": \"%s\"}\n",
           names[mode], ms, (mode & 1) ? ops / (ms * 1e-3) / 1e12 : 0.0,
           (mode & 2) ? bytes / (ms * 1e-3) / 1e12 : 0.0, cudaGetErrorString(cudaGetLastError()));
  }
  {
    // TMA 2D boxes over a [rows, 1152] u8 tensor (L2-resident 9.4 MB)
    const int rows = 8192;
    uint8_t* t;
    cudaMalloc(&t, (size_t)rows * 1152);
    cudaMemset(t, 3, (size_t)rows * 1152);
    if (getenv("PROBE_RANDOM")) {  // random bytes: the MMA's data-dependent power
      uint8_t* h = (uint8_t*)malloc((size_t)rows * 1152);
      uint32_t x = 12345;
      for (size_t i = 0; i < (size_t)rows * 1152; ++i) {
        x = x * 1664525u + 1013904223u;
        h[i] = (uint8_t)(x >> 24);
      }
      cudaMemcpy(t, h, (size_t)rows * 1152, cudaMemcpyHostToDevice);
      free(h);
    }
    CUtensorMap tm;
    cuuint64_t dims[2] = {1152, (cuuint64_t)rows};
    cuuint64_t strides[1] = {1152};
    cuuint32_t box[2] = {128, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, t, dims, strides, box,
                                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    for (int stages = 4; stages <= 6; ++stages) {
      const int sm3 = stages * 32768 + 2 * stages * 8 + 64 + 1024;
      cudaFuncSetAttribute(pipeline_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, sm3);
      pipeline_pair<<<sms, 128, sm3>>>(stages, 450, rows, tm);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      pipeline_pair<<<sms, 128, sm3>>>(stages, 4005, rows, tm);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 2.0 * 256 * 256 * 128 * 4005.0 * (sms / 2);
      printf("{\"mode\": \"CTA-pair pipeline, TMA 2D boxes, %d x 32 KB stages per CTA\", \"ms\": %.3f, \"mma_tops\": %.0f, \"err\": \"%s\"}\n",
             stages, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    for (int stages = 3; stages <= 4; ++stages) {
      const int sm2 = stages * 49152 + 2 * stages * 8 + 64 + 1024;
      cudaFuncSetAttribute(pipeline_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
      pipeline_tma<<<sms, 128, sm2>>>(stages, 450, rows, tm);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      pipeline_tma<<<sms, 128, sm2>>>(stages, 4005, rows, tm);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 2.0 * 128 * 256 * 128 * 4005.0 * sms;
      printf("{\"mode\": \"gemm pipeline, TMA 2D boxes, %d x 48 KB stages\", \"ms\": %.3f, \"mma_tops\": %.0f, \"err\": \"%s\"}\n",
             stages, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int stages = 2; stages <= 4; ++stages) {
    const int sm2 = stages * 49152 + 2 * stages * 8 + 64 + 1024;
    cudaFuncSetAttribute(pipeline, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2);
    pipeline<<<sms, 128, sm2>>>(stages, 400, g, span);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    pipeline<<<sms, 128, sm2>>>(stages, 4000, g, span);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = 2.0 * 128 * 256 * 128 * 4000.0 * sms;
    printf("{\"mode\": \"gemm pipeline, %d x 48 KB stages\", \"ms\": %.3f, \"mma_tops\": %.0f, \"err\": \"%s\"}\n",
           stages, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
