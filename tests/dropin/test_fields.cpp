// Drop-in semantics checks (not a reference test):
//  1. qlinear_forward reads the layer's current fields (qgemm.cpp:23-67 reads
//     w_q, bias and act_bits on every call): after a forward, changing those
//     fields must change the result exactly as a freshly built layer with the
//     same fields would; a copy that diverges from its source must not share
//     the source's device weights.
//  2. Group sizes have no device limit: per_tensor() params over a matrix of
//     more than 16384 elements and per_channel() over many rows follow
//     compute_minmax_params (quant.cpp:90-113) restated here on the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "dtq/qgemm.hpp"
#include "dtq/quant.hpp"

using namespace dtq;

static Matrix random_matrix(std::size_t r, std::size_t c, std::mt19937_64& rng, double scale) {
  std::normal_distribution<double> d(0.0, scale);
  Matrix m(r, c);
  for (auto& v : m.data()) v = d(rng);
  return m;
}

static int failures = 0;
static void expect(bool ok, const char* what) {
  std::printf("%s: %s\n", ok ? "ok  " : "FAIL", what);
  if (!ok) ++failures;
}

static QuantLinear fresh(const QuantLinear& l) { return QuantLinear{l.w_q, l.bias, l.act_bits}; }

int main() {
  std::mt19937_64 rng(5);
  const Matrix w = random_matrix(64, 96, rng, 1.0);
  const Matrix x = random_matrix(21, 96, rng, 2.0);
  QuantLinear layer = make_quant_linear(w, 8, 8, std::vector<double>(64, 0.25));
  const Matrix y0 = qlinear_forward(x, layer);
  QuantLinear copy = layer;  // shares the device handle until it diverges

  layer.bias = std::vector<double>(64, -1.5);
  expect(qlinear_forward(x, layer).data() == qlinear_forward(x, fresh(layer)).data(),
         "bias change after the first forward is seen");
  expect(qlinear_forward(x, copy).data() == y0.data(), "unchanged copy keeps its result");

  layer.w_q.ints[5] = static_cast<uint8_t>(layer.w_q.ints[5] ^ 1);
  layer.w_q.params[3].scale *= 2.0;
  expect(qlinear_forward(x, layer).data() == qlinear_forward(x, fresh(layer)).data(),
         "weight code / scale change is seen");

  layer.act_bits = 4;
  expect(qlinear_forward(x, layer).data() == qlinear_forward(x, fresh(layer)).data(),
         "act_bits change is seen");
  expect(qlinear_forward(x, copy).data() == y0.data(), "copy still unaffected");

  // per-tensor params over 300 x 100 = 30000 elements (> 16384)
  Matrix big = random_matrix(300, 100, rng, 3.0);
  big(7, 9) = 41.0;
  const QuantizedTensor q = quantize(big, GroupingScheme::per_tensor(), 8, QuantMode::Dynamic);
  double mn = big.data()[0], mx = mn;
  for (double v : big.data()) {
    mn = std::min(mn, v);
    mx = std::max(mx, v);
  }
  const double lo = std::min(mn, 0.0), hi = std::max(mx, 0.0), s = (hi - lo) / 255.0;
  const int z = static_cast<int>(std::clamp(round_even(-lo / s), 0.0, 255.0));
  expect(q.params.size() == 1 && q.params[0].scale == s && q.params[0].zero_point == z,
         "per_tensor params over 30000 elements");
  bool codes_ok = true;
  for (std::size_t r = 0; r < big.rows(); ++r)
    for (std::size_t c = 0; c < big.cols(); ++c) {
      const double k = std::clamp(round_even(big(r, c) / s) + z, 0.0, 255.0);
      codes_ok &= q.code(r, c) == static_cast<uint8_t>(k);
    }
  expect(codes_ok, "per_tensor codes over 30000 elements");

  // per-channel params: 20000 rows -> groups of 20000 elements
  Matrix tall = random_matrix(20000, 3, rng, 1.0);
  const QuantizedTensor qc = quantize(tall, GroupingScheme::per_channel(), 6, QuantMode::Dynamic,
                                      nullptr, true);
  bool ch_ok = qc.params.size() == 3;
  for (std::size_t c = 0; c < 3 && ch_ok; ++c) {
    double amax = 0.0;
    for (std::size_t r = 0; r < tall.rows(); ++r) amax = std::max(amax, std::abs(tall(r, c)));
    ch_ok &= qc.params[c].scale == amax / 31.0 && qc.params[c].zero_point == 32;
  }
  expect(ch_ok, "per_channel symmetric params over 20000-row channels");

  std::printf("%s\n", failures == 0 ? "fields ok" : "fields FAILED");
  return failures == 0 ? 0 : 1;
}
