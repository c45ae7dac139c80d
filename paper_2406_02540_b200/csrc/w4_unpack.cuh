// w4_unpack.cuh -- W4A8 weights, packed nibbles -> s8 rows for the W8A8 GEMM.
//
// A W4A8 forward stores its weights as 4-bit codes (the memory the format
// saves) and, per forward, expands them to s8 w = c - 8 in the forward
// workspace: B200 has no int4 MMA, and an L2-resident s8 copy lets the
// W8A8 kernels (CTA pairs, no converter warps) run the GEMM.  The expansion
// rides along the tile quantizer of the same forward (its CTAs take a
// grid-stride share of the chunks after griddepcontrol.wait: the previous
// forward's GEMM may still read the workspace until then), or runs as its
// own kernel in front of the GEMM when another quantizer kernel is used.
//
// Nibble layout (weight_pack_kernel in capi.cu): word i of a row holds
// columns 8i..8i+7, byte k = n[8i+k] | n[8i+k+4] << 4, n = c ^ 8 (the 4-bit
// two's complement of c - 8).  One chunk = 16 packed bytes = 32 columns.
#pragma once

#include <cstdint>

namespace dtq_w4 {

struct Unpack {
  const uint8_t* src;  // [rows, ld4] packed nibbles (nullptr: no job)
  int64_t ld4;
  int64_t rows;           // N
  int64_t chunks;            // 16-byte chunks per row: ceil(round_up(K, 8) / 32)
  int8_t* dst;         // [rows, ld8] s8
  int64_t ld8;               // round_up(K, 16)
};

__device__ __forceinline__ void unpack_range(const Unpack& u, int64_t first, int64_t stride) {
  const int64_t total = u.rows * u.chunks;
  for (int64_t i = first; i < total; i += stride) {
    const int64_t o = i / u.chunks, c = i - o * u.chunks;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(u.src + o * u.ld4) + c);
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
    uint32_t r[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // per byte: (n ^ 8) - 8 sign-extends the nibble n
      r[2 * j] = __vsub4((wv[j] & 0x0F0F0F0Fu) ^ 0x08080808u, 0x08080808u);
      r[2 * j + 1] = __vsub4(((wv[j] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u, 0x08080808u);
    }
    int8_t* d = u.dst + o * u.ld8 + 32 * c;
    *reinterpret_cast<uint4*>(d) = make_uint4(r[0], r[1], r[2], r[3]);
    if (32 * c + 16 < u.ld8) *reinterpret_cast<uint4*>(d + 16) = make_uint4(r[4], r[5], r[6], r[7]);
  }
}

}  // namespace dtq_w4
