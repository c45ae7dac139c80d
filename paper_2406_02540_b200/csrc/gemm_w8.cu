// gemm_w8.cu -- W8A8 instantiations of the tcgen05 GEMM (qgemm_sm100.cuh).
#include "launch.h"

cudaError_t dtq_launch_gemm_w8(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st) {
  // per-CTA smem ring (192 KB): single CTA 4 x (16 KB A + 32 KB B) at BN=256,
  // 6 x (16 + 16) at BN=128; CTA pair 6 x (16 + 16) at BN=256, 8 x (16 + 8) at BN=128
  if (c.cta2)
    return c.bn == 256 ? dtq_launch_gemm_o<256, 6, false, true>(tA, tB, tY, g, sms, st)
                       : dtq_launch_gemm_o<128, 8, false, true>(tA, tB, tY, g, sms, st);
  return c.bn == 256 ? dtq_launch_gemm_o<256, 4, false, false>(tA, tB, tY, g, sms, st)
                     : dtq_launch_gemm_o<128, 6, false, false>(tA, tB, tY, g, sms, st);
}
