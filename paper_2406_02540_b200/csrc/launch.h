// launch.h -- kernel launchers shared by the C-ABI (capi.cu) and the
// per-family kernel translation units (fq_kernels.cu, gemm_w8.cu, gemm_w4.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "fused_quant.cuh"
#include "qgemm_sm100.cuh"

// fused activation / weight quantizer; x_dtype is a dtq_dtype
cudaError_t dtq_launch_fq(const dtq_fq::FqArgs& a, int x_dtype, bool exact, int cpt, bool vec,
                          int block, int sms, cudaStream_t st);

// tcgen05 integer GEMM; BN in {128, 256}
cudaError_t dtq_launch_gemm_w8(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int BN, int sms,
                               cudaStream_t st);
cudaError_t dtq_launch_gemm_w4(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int BN, int sms,
                               cudaStream_t st);

template <int BN, int kStages, bool kW4, int kOut>
cudaError_t dtq_launch_gemm_t(const CUtensorMap& tA, const CUtensorMap& tB,
                              const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int sms,
                              cudaStream_t st) {
  using L = dtq_gemm::Smem<BN, kStages, kW4>;
  auto kern = dtq_gemm::qgemm_kernel<BN, kStages, kW4, kOut>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_dev != dev) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::alloc);
    if (e != cudaSuccess) return e;
    configured_dev = dev;
  }
  const int tiles = g.tiles_m * g.tiles_n;
  const int grid = tiles < sms ? tiles : sms;
  kern<<<grid, dtq_gemm::num_threads<BN, kW4>(), L::alloc, st>>>(tA, tB, tY, g);
  return cudaGetLastError();
}

template <int BN, int kStages, bool kW4>
cudaError_t dtq_launch_gemm_o(const CUtensorMap& tA, const CUtensorMap& tB,
                              const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int sms,
                              cudaStream_t st) {
  switch (g.out_kind) {
    case dtq_gemm::kOutF16:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutF16>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutBF16:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutBF16>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutF32:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutF32>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutS32:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutS32>(tA, tB, tY, g, sms, st);
    default:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutNone>(tA, tB, tY, g, sms, st);
  }
}
