// fq_tile.cu -- instantiations + launcher of the register-resident fused
// quantizer (fused_quant_tile.cuh) for fp16 / bf16 / fp32 input, with and
// without the 128-column rotation.
#include <cstdlib>

#include "fused_quant_tile.cuh"

#include "fq_tile_launch.h"

// Rows per tile: the largest power of two <= 16 with <= 576 threads and the
// CTA in 200 KB of smem (R = 16 at K = 1152: 288 threads, two CTAs per SM;
// R = 8 at K = 4608: 576 threads, one), halved (down to 4) while the grid
// would leave CTA slots idle.  DTQ_FQ_R overrides (diagnostics).
int dtq_fq_tile_rows(int64_t M, int64_t K, int es, bool has_a, bool has_b, int sms) {
  // K <= 2304: four lanes per block, <= 288 threads (R = 8 at K = 1152);
  // wider: two lanes per block, <= 576 threads (R = 8 at K = 4608)
  const int cap = dtq_fq::fq_lanes(K) == 4 ? 288 : 576;
  int R = 16;
  while (R > 1 && (dtq_fq::fq_tile_threads(K, R) > cap ||
                   dtq_fq::fq_tile_layout(K, R, es, has_a, has_b).bytes > 100 * 1024))
    R >>= 1;
  while (R > 4 && (M + R - 1) / R < 2 * sms) R >>= 1;
  static const int forced = [] {
    const char* e = std::getenv("DTQ_FQ_R");
    return e ? std::atoi(e) : 0;
  }();
  if ((forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16) && dtq_fq::fq_tile_threads(K, forced) <= cap)
    R = forced;
  return R;
}

cudaError_t dtq_launch_fq_tile_f16(const dtq_fq::FqArgs& a, bool rot, int R, int sms,
                                   cudaStream_t st);
cudaError_t dtq_launch_fq_tile_bf16(const dtq_fq::FqArgs& a, bool rot, int R, int sms,
                                    cudaStream_t st);

cudaError_t dtq_launch_fq_tile(const dtq_fq::FqArgs& a, int x_dtype_size, int x_is_bf16, bool rot,
                               int R, int sms, cudaStream_t st) {
  if (x_dtype_size == 4) return launch_rot<float>(a, rot, R, sms, st);
  if (x_is_bf16) return dtq_launch_fq_tile_bf16(a, rot, R, sms, st);
  return dtq_launch_fq_tile_f16(a, rot, R, sms, st);
}
