// gemm_w8.cu -- W8A8 instantiations of the tcgen05 GEMM (qgemm_sm100.cuh).
#include "launch.h"

cudaError_t dtq_launch_gemm_w8(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st) {
  // per-CTA smem ring next to the epilogue staging (32 KB double-buffered,
  // 16 KB single for pairs at BN=256): single CTA 3 x (16 KB A + 32 KB B) at
  // BN=256, 5 x (16 + 16) at BN=128; CTA pair 6 x (16 + 16) at BN=256,
  // 7 x (16 + 8) at BN=128
#ifndef DTQ_W8_P256
#define DTQ_W8_P256 6
#endif
  if (c.cta2)
    return c.bn == 256 ? dtq_launch_gemm_o<256, DTQ_W8_P256, false, true>(tA, tB, tY, g, sms, st)
                       : dtq_launch_gemm_o<128, 7, false, true>(tA, tB, tY, g, sms, st);
  return c.bn == 256 ? dtq_launch_gemm_o<256, 3, false, false>(tA, tB, tY, g, sms, st)
                     : dtq_launch_gemm_o<128, 5, false, false>(tA, tB, tY, g, sms, st);
}
