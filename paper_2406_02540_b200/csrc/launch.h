// launch.h -- kernel launchers shared by the C-ABI (capi.cu) and the
// per-family kernel translation units (fq_kernels.cu, gemm_w8.cu, gemm_w4.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include "fused_quant.cuh"
#include "fused_quant_fast.cuh"
#include "qgemm_sm100.cuh"

// fused activation / weight quantizer: fp64 "exact" kernel (x_dtype is a
// dtq_dtype) and the fp32 "fast" kernels per input type
cudaError_t dtq_launch_fq_exact(const dtq_fq::FqArgs& a, int x_dtype, int cpt, bool vec,
                                int block, int sms, cudaStream_t st);
int dtq_fq_tile_rows(int64_t M, int64_t K, int es, bool has_a, bool has_b, int pro, bool exact_v,
                     int sms);
cudaError_t dtq_launch_fq_tile(const dtq_fq::FqArgs& a, int x_dtype_size, int x_is_bf16, bool rot,
                               int R, int sms, cudaStream_t st);
cudaError_t dtq_launch_fq_fast_f16(const dtq_fq::FqArgs& a, int cpt, bool rot, int block, int sms,
                                   cudaStream_t st);
cudaError_t dtq_launch_fq_fast_bf16(const dtq_fq::FqArgs& a, int cpt, bool rot, int block, int sms,
                                    cudaStream_t st);
cudaError_t dtq_launch_fq_fast_f32(const dtq_fq::FqArgs& a, int cpt, bool rot, int block, int sms,
                                   cudaStream_t st);

// tcgen05 integer GEMM tile configurations
struct GemmCfg {
  int bn;    // 128 or 256
  int cta2;  // 1: CTA pair (256-row tiles, cta_group::2)
};
// tcgen05 integer GEMM (W8A8)
cudaError_t dtq_launch_gemm_w8(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st);
cudaError_t dtq_launch_gemm_w4(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st);

// W8A8 tiles that share each SM with the tile quantizer (row flags):
// per-SM registers / shared memory of the instance for (c, out_kind), and the
// launcher (gemm_w8_cores.cu)
int dtq_gemm_w8_cores_info(GemmCfg c, int out_kind, int* regs_per_sm, int* smem);
cudaError_t dtq_launch_gemm_w8_cores(const CUtensorMap& tA, const CUtensorMap& tB,
                                     const CUtensorMap& tY, const dtq_gemm::GemmArgs& g,
                                     GemmCfg c, int sms, cudaStream_t st);

template <int BN, int kStages, bool kW4, int kOut, bool k2Cta, bool kCoRes = false, int kAct = 0>
cudaError_t dtq_launch_gemm_t(const CUtensorMap& tA, const CUtensorMap& tB,
                              const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int sms,
                              cudaStream_t st) {
  using L = dtq_gemm::Smem<BN, kStages, kW4, k2Cta>;
  auto kern = dtq_gemm::qgemm_kernel<BN, kStages, kW4, kOut, k2Cta, kCoRes, kAct>;
  static thread_local int configured_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (configured_dev != dev) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::alloc);
    if (e != cudaSuccess) return e;
#ifndef DTQ_NO_CARVEOUT
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
#endif
    configured_dev = dev;
  }
  const int tiles = g.tiles_m * g.tiles_n;
  const int per = k2Cta ? 2 : 1;                   // CTAs per tile
  const int units = sms / per;
  const int grid = per * (tiles < units ? tiles : units);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dtq_gemm::num_threads<BN, kW4>());
  cfg.dynamicSmemBytes = L::alloc;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = per;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the GEMM's CTAs may start (barrier init,
  // TMEM allocation, descriptor prefetch) while the quantizer that produces
  // its A operand drains; the kernel waits (griddepcontrol.wait) before
  // touching codes / s_x / z_x
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, tA, tB, tY, g);
}

template <int BN, int kStages, bool kW4, bool k2Cta>
cudaError_t dtq_launch_gemm_o(const CUtensorMap& tA, const CUtensorMap& tB,
                              const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int sms,
                              cudaStream_t st) {
  switch (g.out_kind) {
    case dtq_gemm::kOutF16:
      if (g.act == 1)  // GELU epilogue (fp16 / bf16 outputs)
        return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutF16, k2Cta, false, 1>(tA, tB, tY,
                                                                                     g, sms, st);
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutF16, k2Cta>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutBF16:
      if (g.act == 1)
        return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutBF16, k2Cta, false, 1>(tA, tB, tY,
                                                                                      g, sms, st);
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutBF16, k2Cta>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutF32:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutF32, k2Cta>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutS32:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutS32, k2Cta>(tA, tB, tY, g, sms, st);
    default:
      return dtq_launch_gemm_t<BN, kStages, kW4, dtq_gemm::kOutNone, k2Cta>(tA, tB, tY, g, sms, st);
  }
}
