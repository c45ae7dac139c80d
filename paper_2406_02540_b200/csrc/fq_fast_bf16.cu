// fq_fast_bf16.cu -- fp32 fused-quantizer instantiations for __nv_bfloat16 input
// (fused_quant_fast.cuh): without / with the 128-column rotation, for the
// compile-time step counts up to 5 (K <= 1280, e.g. the 1152-wide STDiT /
// PixArt activations) and a runtime-step, multi-warp-per-row fallback.
#include "launch.h"

namespace {

template <bool kRot, int kNit>
cudaError_t launch_t(const dtq_fq::FqArgs& a, int block, int sms, cudaStream_t st) {
  auto kern = dtq_fq::fq_fast_kernel<__nv_bfloat16, kRot, kNit>;
  const int rows_per_cta = block / a.tpr;
  const size_t smem = dtq_fq::fq_fast_smem_bytes(rows_per_cta, a.K, 2);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
  if (e != cudaSuccess) return e;
  const int64_t ctas = (a.M + rows_per_cta - 1) / rows_per_cta;
  const int64_t cap = static_cast<int64_t>(sms) * (occ > 0 ? occ : 1);
  const int grid = static_cast<int>(ctas < cap ? ctas : cap);
  kern<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool kRot>
cudaError_t launch_r(const dtq_fq::FqArgs& a, int nit, int block, int sms, cudaStream_t st) {
  switch (nit) {
    case 1: return launch_t<kRot, 1>(a, block, sms, st);
    case 2: return launch_t<kRot, 2>(a, block, sms, st);
    case 3: return launch_t<kRot, 3>(a, block, sms, st);
    case 4: return launch_t<kRot, 4>(a, block, sms, st);
    case 5: return launch_t<kRot, 5>(a, block, sms, st);
    default: return launch_t<kRot, 0>(a, block, sms, st);
  }
}

}  // namespace

// nit: compile-time step count to use (0 = runtime loop with tpr/32 warps per row)
cudaError_t dtq_launch_fq_fast_bf16(const dtq_fq::FqArgs& a, int nit, bool rot, int block,
                                  int sms, cudaStream_t st) {
  return rot ? launch_r<true>(a, nit, block, sms, st) : launch_r<false>(a, nit, block, sms, st);
}
