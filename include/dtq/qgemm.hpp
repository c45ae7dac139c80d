// dtq/qgemm.hpp -- drop-in interface mirror of the reference quantized
// linear (/root/reference/proj/core/include/dtq/qgemm.hpp:17-54).
// make_quant_linear prepares the weights on the B200 and keeps them resident
// (opaque handle in QuantLinear::device); qlinear_forward runs the fused
// quantizer + tcgen05 integer GEMM and the reference's fp64 epilogue, so its
// output is bit-identical to the reference.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <utility>
#include <vector>

#include "dtq/matrix.hpp"
#include "dtq/quant.hpp"

namespace dtq {

struct QuantLinear {
  QuantizedTensor w_q;                      // [C_out, C_in], PerOutputChannel, symmetric
  std::optional<std::vector<double>> bias;  // length C_out
  int act_bits = 8;
  // device-resident prepared weights (built lazily for hand-made layers)
  mutable std::shared_ptr<void> device;

  std::size_t out_channels() const { return w_q.rows; }
  std::size_t in_channels() const { return w_q.cols; }
};

QuantLinear make_quant_linear(const Matrix& w, int weight_bits, int act_bits,
                              const std::optional<std::vector<double>>& bias = {});
Matrix qlinear_forward(const Matrix& x, const QuantLinear& layer);
Matrix qlinear_forward_float(const Matrix& x, const QuantLinear& layer);

struct LayerBytes {
  std::size_t weights = 0;
  std::size_t params = 0;
};
LayerBytes weight_bytes(std::size_t rows, std::size_t cols, int bits, std::size_t group_count);
std::size_t checkpoint_bytes(const std::vector<std::pair<Matrix, int>>& layers);
std::size_t fp16_baseline_bytes(const std::vector<std::pair<Matrix, int>>& layers);

}  // namespace dtq
