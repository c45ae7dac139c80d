// fq_fast_f16.cu -- fp32 fused-quantizer instantiations for __half input
// (fused_quant_fast.cuh): without / with the 128-column rotation, for
// G = 1, 2, 4 lane groups (of 8 lanes) per row.
#include "launch.h"

namespace {

template <bool kRot, int G, int kNblk>
cudaError_t launch_t(const dtq_fq::FqArgs& a, int block, int sms, cudaStream_t st) {
  auto kern = dtq_fq::fq_fast_kernel<__half, kRot, G, kNblk>;
  const int warps = block / 32;
  const size_t smem = warps * dtq_fq::fq_fast_warp_bytes(a.K, G, 2);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  int occ = 0;
  const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
  if (e != cudaSuccess) return e;
  const int rows_per_cta = warps * (4 / G);
  const int64_t ctas = (a.M + rows_per_cta - 1) / rows_per_cta;
  const int64_t cap = static_cast<int64_t>(sms) * (occ > 0 ? occ : 1);
  const int grid = static_cast<int>(ctas < cap ? ctas : cap);
  kern<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool kRot, int G>
cudaError_t launch_k(const dtq_fq::FqArgs& a, int block, int sms, cudaStream_t st) {
  // (compile-time-K instantiations measured slower: full unrolling bloats
  // the code; the runtime-K loop is used for every width)
  return launch_t<kRot, G, 0>(a, block, sms, st);
}

template <bool kRot>
cudaError_t launch_r(const dtq_fq::FqArgs& a, int G, int block, int sms, cudaStream_t st) {
  switch (G) {
    case 1: return launch_k<kRot, 1>(a, block, sms, st);
    case 2: return launch_k<kRot, 2>(a, block, sms, st);
    default: return launch_k<kRot, 4>(a, block, sms, st);
  }
}

}  // namespace

// G: 8-lane groups per row (1, 2 or 4)
cudaError_t dtq_launch_fq_fast_f16(const dtq_fq::FqArgs& a, int G, bool rot, int block,
                                  int sms, cudaStream_t st) {
  return rot ? launch_r<true>(a, G, block, sms, st) : launch_r<false>(a, G, block, sms, st);
}
