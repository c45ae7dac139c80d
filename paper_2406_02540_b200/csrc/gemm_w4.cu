// gemm_w4.cu -- W4A8 instantiations (packed nibbles unpacked in smem).
#include "launch.h"

cudaError_t dtq_launch_gemm_w4(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int BN, int sms,
                               cudaStream_t st) {
  // smem ring: 3 x (16 KB A + 16 KB packed + 32 KB s8) at BN=256
  return BN == 256 ? dtq_launch_gemm_o<256, 3, true, false>(tA, tB, tY, g, sms, st)
                   : dtq_launch_gemm_o<128, 4, true, false>(tA, tB, tY, g, sms, st);
}
