// int8_ceiling.cu -- the dense INT8 tensor-core ceiling of this B200
// (diagnostics).  One persistent CTA per SM (or
// CTA pair) issues tcgen05.mma.kind::i8 (u8 x s8 -> s32, the GEMM's exact
// instruction and descriptors) back to back from operands resident in shared
// memory: no TMA, no epilogue, no HBM traffic -- the rate at which the
// tensor pipe retires the qgemm kernel's MMAs.  Times a short burst (~100 us,
// under the power cap) and a sustained run (~20 ms) with CUDA events.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//          -I../paper_2406_02540_b200/csrc int8_ceiling.cu -o _bin/int8_ceiling -lcuda
// usage: int8_ceiling   (prints one JSON line)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace dtq_ptx;

template <int BN, bool k2Cta>
__global__ void __launch_bounds__(128, 1) mma_peak_kernel(int iters, unsigned long long* sink) {
  constexpr int BM = 128, BK = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;                          // 128 x 128 B
  uint8_t* sB = smem + BM * BK;                // (BN or BN/2) x 128 B
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (k2Cta ? BN / 2 : BN) * BK);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const uint32_t rank = k2Cta ? cluster_ctarank() : 0;
  // operands: uniformly random bytes, like real codes and weights (the rate
  // DOES depend on the values: the tensor cores' power, hence the clock, does;
  // a low-toggle pattern reads ~15 % faster)
  uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int i = threadIdx.x; i < (BM + (k2Cta ? BN / 2 : BN)) * BK / 16; i += blockDim.x) {
    uint32_t w[4];
    for (int j = 0; j < 4; ++j) {
      x = x * 1664525u + 1013904223u;
      w[j] = x ^ (x >> 15);
    }
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) {
    if constexpr (k2Cta)
      tmem_alloc_cta2<2 * BN>(slot);
    else
      tmem_alloc<2 * BN>(slot);
  }
  tc_fence_before();
  if constexpr (k2Cta)
    cluster_sync();
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  constexpr uint32_t idesc = idesc_i8_u8s8(k2Cta ? 2 * BM : BM, BN);
  if (threadIdx.x == 0 && rank == 0) {
    const uint64_t ad = umma_desc_sw128(smem_u32(sA)), bd = umma_desc_sw128(smem_u32(sB));
    for (int it = 0; it < iters; ++it) {
      // one 128-byte k-block = 4 x K=32 MMAs, alternating TMEM accumulators
      const uint32_t d = tmem + (it & 1) * BN;
#pragma unroll
      for (int k = 0; k < BK / 32; ++k) {
        if constexpr (k2Cta)
          mma_i8_cta2(d, ad + 2 * k, bd + 2 * k, idesc, k != 0 ? 1u : 0u);
        else
          mma_i8(d, ad + 2 * k, bd + 2 * k, idesc, k != 0 ? 1u : 0u);
      }
    }
    if constexpr (k2Cta)
      mma_commit_cta2_mc(bar, 0x3);
    else
      mma_commit(bar);
  }
  if (threadIdx.x == 0) {
    mbar_wait(bar, 0);
    if (blockIdx.x == 0) sink[0] = tmem;
  }
  tc_fence_before();
  if constexpr (k2Cta)
    cluster_sync();
  else
    __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    if constexpr (k2Cta)
      tmem_dealloc_cta2<2 * BN>(tmem);
    else
      tmem_dealloc<2 * BN>(tmem);
  }
}

template <int BN, bool k2Cta>
double run(int sms, int iters, int reps, double* ms_out) {
  auto kern = mma_peak_kernel<BN, k2Cta>;
  const int smem = 128 * 128 + (k2Cta ? BN / 2 : BN) * 128 + 64 + 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sms - (k2Cta ? sms % 2 : 0));
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = k2Cta ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, iters, sink);  // warm-up
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, kern, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "launch failed: %s\n", cudaGetErrorString(e));
    return 0.0;
  }
  const int units = k2Cta ? cfg.gridDim.x / 2 : cfg.gridDim.x;
  const double mrows = k2Cta ? 256.0 : 128.0;
  const double ops = 2.0 * mrows * BN * 128.0 * iters * units * reps;
  *ms_out = ms / reps;
  cudaFree(sink);
  return ops / (ms * 1e-3) / 1e12;
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double ms1 = 0, ms2 = 0, ms3 = 0, ms4 = 0;
  // burst: ~100 us per launch (below the power-cap response)
  const double b1 = run<256, false>(sms, 400, 5, &ms1);
  const double b2 = run<256, true>(sms, 400, 5, &ms2);
  // sustained: ~20 ms of back-to-back launches
  const double s1 = run<256, false>(sms, 4000, 20, &ms3);
  const double s2 = run<256, true>(sms, 4000, 20, &ms4);
  printf("{\"int8_ceiling_burst_tops_1cta\": %.1f, \"int8_ceiling_burst_tops_2cta\": %.1f, "
         "\"int8_ceiling_sustained_tops_1cta\": %.1f, \"int8_ceiling_sustained_tops_2cta\": %.1f, "
         "\"burst_launch_us\": %.1f, \"sms\": %d, \"sm_clock_mhz_nominal\": %d, "
         "\"nominal_tops_at_nominal_clock\": 4500, \"what\": \"tcgen05.mma.kind::i8 u8xs8->s32 "
         "M=128|256 N=256 K=32 back to back from smem, random operands, no TMA/epilogue\"}\n",
         b1, b2, s1, s2, ms1 * 1e3, sms, clk_khz / 1000);
  return 0;
}
