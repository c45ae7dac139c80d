// fq_tile.cu -- instantiations + launcher of the register-resident fused
// quantizer (fused_quant_tile.cuh) for fp16 / bf16 / fp32 input, with and
// without the 128-column rotation.
#include <cstdlib>

#include "fused_quant_tile.cuh"

namespace {

template <typename Tin, bool kRot, bool kExactV, int kPro>
cudaError_t launch_tile(const dtq_fq::FqArgs& a, int R, int sms, cudaStream_t st) {
  auto kern = dtq_fq::fq_tile_kernel<Tin, kRot, kExactV, kPro>;
  const bool has_b = a.pro == dtq_fq::kProModulate || a.pro == dtq_fq::kProLnModulate;
  const bool has_a = has_b || a.col_mul != nullptr;
  const dtq_fq::TileLayout L = dtq_fq::fq_tile_layout(a.K, R, sizeof(Tin), has_a, has_b);
  const int nb = static_cast<int>(a.K / 128);
  const int block = dtq_fq::fq_tile_threads(a.K, R);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(L.bytes));
  if (e != cudaSuccess) return e;
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, L.bytes);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.M + R - 1) / R;
  const int64_t cap = static_cast<int64_t>(sms) * (occ > 0 ? occ : 1);
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  kern<<<grid, block, L.bytes, st>>>(a, R);
  return cudaGetLastError();
}

template <typename Tin, int kPro>
cudaError_t launch_p(const dtq_fq::FqArgs& a, bool rot, int R, int sms, cudaStream_t st) {
  if (rot) return launch_tile<Tin, true, false, kPro>(a, R, sms, st);
  if constexpr (kPro == dtq_fq::kProNone) {
    // no prologue, smoothing or rotation: codes are reachable bit for bit
    if (a.col_mul == nullptr) return launch_tile<Tin, false, true, kPro>(a, R, sms, st);
  }
  return launch_tile<Tin, false, false, kPro>(a, R, sms, st);
}

template <typename Tin>
cudaError_t launch_rot(const dtq_fq::FqArgs& a, bool rot, int R, int sms, cudaStream_t st) {
  switch (a.pro) {
    case dtq_fq::kProModulate: return launch_p<Tin, dtq_fq::kProModulate>(a, rot, R, sms, st);
    case dtq_fq::kProGelu: return launch_p<Tin, dtq_fq::kProGelu>(a, rot, R, sms, st);
    case dtq_fq::kProLnModulate: return launch_p<Tin, dtq_fq::kProLnModulate>(a, rot, R, sms, st);
    default: return launch_p<Tin, dtq_fq::kProNone>(a, rot, R, sms, st);
  }
}

}  // namespace

// Rows per tile: the largest power of two <= 16 with <= 576 threads and the
// CTA in 200 KB of smem (R = 16 at K = 1152: 288 threads, two CTAs per SM;
// R = 8 at K = 4608: 576 threads, one), halved (down to 4) while the grid
// would leave CTA slots idle.  DTQ_FQ_R overrides (diagnostics).
int dtq_fq_tile_rows(int64_t M, int64_t K, int es, bool has_a, bool has_b, int sms) {
  const int64_t nb = K / 128;
  int R = 16;
  while (R > 1 && (dtq_fq::fq_tile_threads(K, R) > 576 ||
                   dtq_fq::fq_tile_layout(K, R, es, has_a, has_b).bytes > 200 * 1024))
    R >>= 1;
  while (R > 4 && (M + R - 1) / R < 2 * sms) R >>= 1;
  static const int forced = [] {
    const char* e = std::getenv("DTQ_FQ_R");
    return e ? std::atoi(e) : 0;
  }();
  if ((forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16) && dtq_fq::fq_tile_threads(K, forced) <= 576)
    R = forced;
  return R;
}

cudaError_t dtq_launch_fq_tile(const dtq_fq::FqArgs& a, int x_dtype_size, int x_is_bf16, bool rot,
                               int R, int sms, cudaStream_t st) {
  if (x_dtype_size == 4) return launch_rot<float>(a, rot, R, sms, st);
  if (x_is_bf16) return launch_rot<__nv_bfloat16>(a, rot, R, sms, st);
  return launch_rot<__half>(a, rot, R, sms, st);
}
