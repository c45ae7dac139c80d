// gemm_w8_cores.cu -- W8A8 GEMM instantiations that run CONCURRENTLY with the
// tile quantizer producing their A operand (row flags, see GemmArgs::ready):
// one quantizer CTA and one GEMM CTA share every SM, so these tiles use a
// shorter stage ring and are capped at 112 registers (qgemm_kernel's kCoRes):
// 320 threads x 112 registers + 288 quantizer threads x 96 registers fit the
// SM's 64K registers.
#include <map>
#include <mutex>
#include <tuple>

#include "launch.h"

namespace {

template <int BN, int kStages, bool k2Cta>
const void* kernel_for(int out_kind) {
  switch (out_kind) {
    case dtq_gemm::kOutF16:
      return reinterpret_cast<const void*>(
          dtq_gemm::qgemm_kernel<BN, kStages, false, dtq_gemm::kOutF16, k2Cta, true>);
    case dtq_gemm::kOutBF16:
      return reinterpret_cast<const void*>(
          dtq_gemm::qgemm_kernel<BN, kStages, false, dtq_gemm::kOutBF16, k2Cta, true>);
    default:
      return reinterpret_cast<const void*>(
          dtq_gemm::qgemm_kernel<BN, kStages, false, dtq_gemm::kOutF32, k2Cta, true>);
  }
}

template <int BN, int kStages, bool k2Cta>
cudaError_t launch(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tY,
                   const dtq_gemm::GemmArgs& g, int sms, cudaStream_t st) {
  switch (g.out_kind) {
    case dtq_gemm::kOutF16:
      return dtq_launch_gemm_t<BN, kStages, false, dtq_gemm::kOutF16, k2Cta, true>(tA, tB, tY, g, sms, st);
    case dtq_gemm::kOutBF16:
      return dtq_launch_gemm_t<BN, kStages, false, dtq_gemm::kOutBF16, k2Cta, true>(tA, tB, tY, g, sms, st);
    default:
      return dtq_launch_gemm_t<BN, kStages, false, dtq_gemm::kOutF32, k2Cta, true>(tA, tB, tY, g, sms, st);
  }
}

}  // namespace

// co-resident stage counts: pairs 4 x 32 KB (BN=256) / 5 x 24 KB (BN=128),
// single CTAs 2 x 48 KB (BN=256) / 4 x 32 KB (BN=128)
#define DTQ_CORES_TILES(X)      \
  X(256, 4, true)               \
  X(128, 5, true)               \
  X(256, 2, false)              \
  X(128, 4, false)

int dtq_gemm_w8_cores_info(GemmCfg c, int out_kind, int* regs_per_sm, int* smem) {
  // cached: cudaFuncGetAttributes costs host microseconds per forward
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, std::pair<int, int>> cache;
  const auto key = std::make_tuple(c.bn, c.cta2, out_kind);
  {
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) {
      *regs_per_sm = it->second.first;
      *smem = it->second.second;
      return 0;
    }
  }
  const void* k = nullptr;
  size_t sm = 0;
#define DTQ_X(BN, S, P)                                              \
  if (c.bn == BN && (c.cta2 != 0) == P) {                           \
    k = kernel_for<BN, S, P>(out_kind);                             \
    sm = dtq_gemm::Smem<BN, S, false, P>::alloc;                    \
  }
  DTQ_CORES_TILES(DTQ_X)
#undef DTQ_X
  if (!k) return -1;
  cudaFuncAttributes at{};
  if (cudaFuncGetAttributes(&at, k) != cudaSuccess) return -1;
  const int threads = dtq_gemm::num_threads<256, false>();
  *regs_per_sm = (at.numRegs + 7) / 8 * 8 * threads;
  *smem = static_cast<int>(sm + at.sharedSizeBytes) + 1024;  // + the CTA's reserved KB
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = std::make_pair(*regs_per_sm, *smem);
  return 0;
}

cudaError_t dtq_launch_gemm_w8_cores(const CUtensorMap& tA, const CUtensorMap& tB,
                                     const CUtensorMap& tY, const dtq_gemm::GemmArgs& g,
                                     GemmCfg c, int sms, cudaStream_t st) {
#define DTQ_X(BN, S, P) \
  if (c.bn == BN && (c.cta2 != 0) == P) return launch<BN, S, P>(tA, tB, tY, g, sms, st);
  DTQ_CORES_TILES(DTQ_X)
#undef DTQ_X
  return cudaErrorInvalidValue;
}
