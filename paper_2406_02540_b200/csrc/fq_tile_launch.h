// fq_tile_launch.h -- launcher template of the tile quantizer, shared by the
// per-dtype translation units (fq_tile.cu, fq_tile_f16.cu, fq_tile_bf16.cu).
#pragma once
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "fused_quant_tile.cuh"

namespace {  // NOLINT

// Launch attributes and occupancy per (kernel, device, block, smem): the
// occupancy query costs microseconds of host time, more than a small launch
// takes on the GPU, so it is made once.
inline cudaError_t fq_tile_occupancy(const void* kern, int block, size_t smem, int* occ) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, size_t>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> smem_max;  // attribute only grows
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const auto key = std::make_tuple(kern, dev, block, smem);
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cache.find(key);
  if (it != cache.end()) {
    *occ = it->second;
    return cudaSuccess;
  }
  size_t& mx = smem_max[std::make_pair(kern, dev)];
  if (smem > mx) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    // the whole unified L1 / shared array as shared memory: an SM running
    // this kernel can then also host the co-resident GEMM CTA (the carveout
    // is fixed while any CTA is resident on the SM)
#ifndef DTQ_NO_CARVEOUT
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
#endif
    mx = smem;
  }
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, kern, block, smem);
  if (e != cudaSuccess) return e;
  cache[key] = *occ;
  return cudaSuccess;
}

// Registers per thread of a kernel (cached; cudaFuncGetAttributes costs
// host microseconds)
inline int fq_kernel_regs(const void* kern) {
  static std::mutex mu;
  static std::map<const void*, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  const auto it = cache.find(kern);
  if (it != cache.end()) return it->second;
  cudaFuncAttributes at{};
  const int r = cudaFuncGetAttributes(&at, kern) == cudaSuccess ? at.numRegs : 255;
  cache[kern] = r;
  return r;
}

template <typename Tin, bool kRot, bool kExactV, int kPro>
cudaError_t launch_tile(const dtq_fq::FqArgs& a_in, int R, int nbuf, int sms, cudaStream_t st) {
  dtq_fq::FqArgs a = a_in;
  // K <= 1152: 4 lanes per block, 8-row tiles (288 threads); wider: 2 lanes
  // per block, 8 or 4 rows (576 threads)
  const bool wide = dtq_fq::fq_lanes(a.K, a.pro) == 2;
  auto kern = !wide ? dtq_fq::fq_tile_kernel<Tin, kRot, kExactV, kPro, false, 8>
              : (R == 8 ? dtq_fq::fq_tile_kernel<Tin, kRot, kExactV, kPro, true, 8>
                        : dtq_fq::fq_tile_kernel<Tin, kRot, kExactV, kPro, true, 4>);
  const bool has_b = a.pro == dtq_fq::kProModulate || a.pro == dtq_fq::kProLnModulate;
  const bool has_a = has_b || a.col_mul != nullptr;
  const dtq_fq::TileLayout L = dtq_fq::fq_tile_layout(a.K, R, sizeof(Tin), has_a, has_b, nbuf);
  const int block = dtq_fq::fq_tile_threads(a.K, R, a.pro);
  int occ = 0;
  cudaError_t e = fq_tile_occupancy(reinterpret_cast<const void*>(kern), block, L.bytes, &occ);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (a.M + R - 1) / R;
  static const int occ_cap = [] {  // DTQ_FQ_OCC (diagnostics): CTAs per SM cap
    const char* e = std::getenv("DTQ_FQ_OCC");
    return e ? std::atoi(e) : 0;
  }();
  if (occ_cap > 0 && occ > occ_cap) occ = occ_cap;
  if (a.ready != nullptr) {
    // row flags: one quantizer CTA per SM next to one GEMM CTA, which runs
    // concurrently and consumes the rows as they are published.  Both must
    // fit an SM together (64K registers in 256-register warp granules; 228 KB
    // of shared memory with 1 KB reserved per CTA, 1 KB of static smem here;
    // partner_smem includes the GEMM's reserved KB), else no flags.
    const int regs = (fq_kernel_regs(reinterpret_cast<const void*>(kern)) + 7) / 8 * 8;
    const int64_t fq_regs = static_cast<int64_t>(regs) * ((block + 31) / 32 * 32);
    const bool fits = fq_regs + a.partner_regs <= 65536 &&
                      static_cast<int64_t>(L.bytes) + 2048 + a.partner_smem <= 228 * 1024;
    if (fits) {
      occ = 1;
    } else {
      a.ready = nullptr;
    }
  }
  if (a.flags_used) *a.flags_used = a.ready != nullptr ? 1 : 0;
  if (a.w4_done) *a.w4_done = a.w4.src != nullptr ? 1 : 0;
  const int64_t cap = static_cast<int64_t>(sms) * (occ > 0 ? occ : 1);
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  // programmatic dependent launch: the CTAs' setup (barriers, the per-column
  // table) overlaps the tail of the kernel that produces X; the kernel waits
  // (griddepcontrol.wait) before its first read of X or of per-call inputs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <typename Tin, int kPro>
cudaError_t launch_p(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms, cudaStream_t st) {
  if (rot) return launch_tile<Tin, true, false, kPro>(a, R, nbuf, sms, st);
  if constexpr (kPro == dtq_fq::kProNone) {
    // no prologue, smoothing or rotation: codes are reachable bit for bit
    if (a.col_mul == nullptr) return launch_tile<Tin, false, true, kPro>(a, R, nbuf, sms, st);
  }
  return launch_tile<Tin, false, false, kPro>(a, R, nbuf, sms, st);
}

template <typename Tin>
cudaError_t launch_rot(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms, cudaStream_t st) {
  switch (a.pro) {
    case dtq_fq::kProModulate: return launch_p<Tin, dtq_fq::kProModulate>(a, rot, R, nbuf, sms, st);
    case dtq_fq::kProGelu: return launch_p<Tin, dtq_fq::kProGelu>(a, rot, R, nbuf, sms, st);
    case dtq_fq::kProLnModulate: return launch_p<Tin, dtq_fq::kProLnModulate>(a, rot, R, nbuf, sms, st);
    default: return launch_p<Tin, dtq_fq::kProNone>(a, rot, R, nbuf, sms, st);
  }
}

}  // namespace
