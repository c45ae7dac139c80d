// gemm_w4.cu -- W4A8 instantiations (packed nibbles unpacked to s8 in smem).
#include "launch.h"

cudaError_t dtq_launch_gemm_w4(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, GemmCfg c,
                               int sms, cudaStream_t st) {
  // unpacked s8 B tiles in a 3-deep ring of their own; the TMA stage ring
  // holds A only (the converter warps read the packed nibbles from L2)
  // (8 epilogue warps double the staging buffers: one stage fewer at BN=256)
// single-CTA stage counts: A + packed nibbles per stage on the TMA path
#ifndef DTQ_W4_S256
#define DTQ_W4_S256 (dtq_gemm::kW4TmaPacked ? 4 : 6)
#endif
#ifndef DTQ_W4_S128
#define DTQ_W4_S128 \
  (dtq_gemm::dual_m<128, true, false>() ? 4 : (dtq_gemm::kW4TmaPacked ? 6 : 9))
#endif
#ifndef DTQ_W4_P256
#define DTQ_W4_P256 (dtq_gemm::kW4TmaPacked ? 6 : 8)
#endif
#ifndef DTQ_W4_P128
#define DTQ_W4_P128 (dtq_gemm::kW4TmaPacked ? 7 : 8)
#endif
  constexpr int kS256 = DTQ_W4_S256, kS128 = DTQ_W4_S128, kP256 = DTQ_W4_P256;
  if (c.cta2)  // CTA pair: each SM unpacks only its half of B (8 A stages fit)
    return c.bn == 256 ? dtq_launch_gemm_o<256, kP256, true, true>(tA, tB, tY, g, sms, st)
                       : dtq_launch_gemm_o<128, DTQ_W4_P128, true, true>(tA, tB, tY, g, sms, st);
  // single CTA: the stage ring holds A only (converters read packed B from L2)
  return c.bn == 256 ? dtq_launch_gemm_o<256, kS256, true, false>(tA, tB, tY, g, sms, st)
                     : dtq_launch_gemm_o<128, kS128, true, false>(tA, tB, tY, g, sms, st);
}
