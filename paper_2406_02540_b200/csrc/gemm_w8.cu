// gemm_w8.cu -- W8A8 instantiations of the tcgen05 GEMM (qgemm_sm100.cuh).
#include "launch.h"

cudaError_t dtq_launch_gemm_w8(const CUtensorMap& tA, const CUtensorMap& tB,
                               const CUtensorMap& tY, const dtq_gemm::GemmArgs& g, int BN, int sms,
                               cudaStream_t st) {
  // smem ring: 4 x (16 KB A + 32 KB B) at BN=256, 6 x (16 + 16) KB at BN=128
  return BN == 256 ? dtq_launch_gemm_o<256, 4, false>(tA, tB, tY, g, sms, st)
                   : dtq_launch_gemm_o<128, 6, false>(tA, tB, tY, g, sms, st);
}
