// fq_tile_bf16.cu -- tile quantizer instantiations for __nv_bfloat16 input.
#include "fq_tile_launch.h"

cudaError_t dtq_launch_fq_tile_bf16(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms,
                                   cudaStream_t st) {
  return launch_rot<__nv_bfloat16>(a, rot, R, nbuf, sms, st);
}
