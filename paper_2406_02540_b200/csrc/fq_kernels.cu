// fq_kernels.cu -- instantiations of the fp64 ("exact") fused quantizer
// (fused_quant.cuh): input {f16, bf16, f32, f64} x {1, 8} chunks per thread
// x {128-bit vector, scalar} loads.  The fp32 ("fast") kernels are in
// fq_fast_*.cu.
#include "../../include/dtq_capi.h"
#include "launch.h"

namespace {

template <typename Tin, int kCPT, bool kVec>
cudaError_t launch_exact_t(const dtq_fq::FqArgs& a, int block, int sms, cudaStream_t st) {
  auto kern = dtq_fq::fq_kernel<Tin, double, kCPT, kVec>;
  static thread_local int occ_cache[33] = {0};
  const int slot = block / 32;
  if (occ_cache[slot] == 0) {
    int occ = 0;
    const cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, 0);
    if (e != cudaSuccess) return e;
    occ_cache[slot] = occ > 0 ? occ : 1;
  }
  const int64_t cap = static_cast<int64_t>(sms) * occ_cache[slot];
  const int grid = static_cast<int>(a.M < cap ? a.M : cap);
  kern<<<grid, block, 0, st>>>(a);
  return cudaGetLastError();
}

template <typename Tin>
cudaError_t launch_exact_c(const dtq_fq::FqArgs& a, int cpt, bool vec, int block, int sms,
                           cudaStream_t st) {
  if (cpt == 1)
    return vec ? launch_exact_t<Tin, 1, true>(a, block, sms, st)
               : launch_exact_t<Tin, 1, false>(a, block, sms, st);
  return vec ? launch_exact_t<Tin, 8, true>(a, block, sms, st)
             : launch_exact_t<Tin, 8, false>(a, block, sms, st);
}

}  // namespace

cudaError_t dtq_launch_fq_exact(const dtq_fq::FqArgs& a, int x_dtype, int cpt, bool vec,
                                int block, int sms, cudaStream_t st) {
  switch (x_dtype) {
    case DTQ_F16: return launch_exact_c<__half>(a, cpt, vec, block, sms, st);
    case DTQ_BF16: return launch_exact_c<__nv_bfloat16>(a, cpt, vec, block, sms, st);
    case DTQ_F32: return launch_exact_c<float>(a, cpt, vec, block, sms, st);
    default: return launch_exact_c<double>(a, cpt, vec, block, sms, st);
  }
}
