// gemm_w4.cu -- W4A8 instantiations (packed nibbles unpacked in smem).
#include "launch.h"

cudaError_t dtq_launch_gemm_w4(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st) {
  // TMA ring per stage: 16 KB A + packed nibbles of this CTA's B rows;
  // unpacked s8 B tiles in a separate 3-deep ring
  if (c.cta2)  // CTA pair: each SM unpacks only its half of B
    return c.bn == 256 ? dtq_launch_gemm_o<256, 6, true, true>(tA, tB, tY, g, sms, st)
                       : dtq_launch_gemm_o<128, 8, true, true>(tA, tB, tY, g, sms, st);
  return c.bn == 256 ? dtq_launch_gemm_o<256, 3, true, false>(tA, tB, tY, g, sms, st)
                     : dtq_launch_gemm_o<128, 6, true, false>(tA, tB, tY, g, sms, st);
}
