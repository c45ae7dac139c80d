// fq_tile.cu -- instantiations + launcher of the register-resident fused
// quantizer (fused_quant_tile.cuh) for fp16 / bf16 / fp32 input, with and
// without the 128-column rotation.
#include <cstdlib>

#include "fused_quant_tile.cuh"

#include "fq_tile_launch.h"

// Rows per tile (compile-time in the kernel): 8, or 4 when an 8-row double
// buffer of a wide row does not fit shared memory.  0 = the shape does not
// fit the tile kernel at all (the caller uses the lane-group kernel).
int dtq_fq_tile_rows(int64_t M, int64_t K, int es, bool has_a, bool has_b, int pro, bool exact_v,
                     int sms) {
  (void)M;
  (void)sms;
  constexpr size_t kMax = 220 * 1024;
  const bool four = dtq_fq::fq_lanes(K, pro) == 4;
  const int cap = four ? 288 : 576;  // the kernels' launch bounds
  static const int force = [] {  // DTQ_FQ_ROWS (diagnostics): start the search at R
    const char* e = std::getenv("DTQ_FQ_ROWS");
    return e ? std::atoi(e) : 8;
  }();
  // wide rows with exact codes (no prologue, smoothing or rotation): 4-row
  // tiles, two 288-thread CTAs per SM instead of one of 576 (the exact-code
  // path's registers spill at 576 threads): 73.7 vs 82.9 us at 16384 x 4608
  const int start = (!four && exact_v && force == 8) ? 4 : force;
  for (int R = start; R >= 4; R /= 2)
    if ((four ? R == 8 : R >= 4) && dtq_fq::fq_tile_threads(K, R, pro) <= cap &&
        dtq_fq::fq_tile_layout(K, R, es, has_a, has_b, 2).bytes <= kMax)
      return R;
  return 0;
}

cudaError_t dtq_launch_fq_tile_f16(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms,
                                   cudaStream_t st);
cudaError_t dtq_launch_fq_tile_bf16(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms,
                                    cudaStream_t st);

cudaError_t dtq_launch_fq_tile(const dtq_fq::FqArgs& a, int x_dtype_size, int x_is_bf16, bool rot,
                               int R, int sms, cudaStream_t st) {
  const int nbuf = 2;  // input double buffer (deeper rings measured no faster)
  if (x_dtype_size == 4) return launch_rot<float>(a, rot, R, nbuf, sms, st);
  if (x_is_bf16) return dtq_launch_fq_tile_bf16(a, rot, R, nbuf, sms, st);
  return dtq_launch_fq_tile_f16(a, rot, R, nbuf, sms, st);
}
