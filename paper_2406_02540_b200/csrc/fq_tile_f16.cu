// fq_tile_f16.cu -- tile quantizer instantiations for __half input.
#include "fq_tile_launch.h"

cudaError_t dtq_launch_fq_tile_f16(const dtq_fq::FqArgs& a, bool rot, int R, int nbuf, int sms,
                                   cudaStream_t st) {
  return launch_rot<__half>(a, rot, R, nbuf, sms, st);
}
