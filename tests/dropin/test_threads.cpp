// Concurrency check of the drop-in (not a reference test): the reference's
// qlinear_forward is a pure function on a const layer, so concurrent calls on
// one layer -- including the first, which uploads it to the device -- must
// give the single-threaded result bit for bit.
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "dtq/qgemm.hpp"

using namespace dtq;

static Matrix random_matrix(std::size_t r, std::size_t c, std::mt19937_64& rng, double scale) {
  std::normal_distribution<double> d(0.0, scale);
  Matrix m(r, c);
  for (auto& v : m.data()) v = d(rng);
  return m;
}

int main() {
  std::mt19937_64 rng(11);
  int failures = 0;
  for (int wbits : {8, 4}) {
    const Matrix w = random_matrix(96, 200, rng, 1.0);
    const QuantLinear made = make_quant_linear(w, wbits, 8);
    // a copy without the device handle: the first forward uploads it lazily
    QuantLinear layer{made.w_q, made.bias, made.act_bits};
    std::vector<Matrix> xs;
    for (int t = 0; t < 8; ++t) xs.push_back(random_matrix(37 + 5 * t, 200, rng, 2.0));
    std::vector<Matrix> ref;
    for (const Matrix& x : xs) ref.push_back(qlinear_forward(x, made));
    std::vector<int> bad(8, 0);
    std::vector<std::thread> pool;
    for (int t = 0; t < 8; ++t)
      pool.emplace_back([&, t] {
        for (int it = 0; it < 25; ++it) {
          const Matrix y = qlinear_forward(xs[t], (it & 1) ? layer : made);
          if (y.data() != ref[t].data()) ++bad[t];
        }
      });
    for (auto& th : pool) th.join();
    for (int t = 0; t < 8; ++t) failures += bad[t];
    std::printf("W%dA8: %d mismatching results over 8 threads x 25 calls\n", wbits,
                [&] { int s = 0; for (int b : bad) s += b; return s; }());
  }
  std::printf("%s\n", failures == 0 ? "threads ok" : "threads FAILED");
  return failures == 0 ? 0 : 1;
}
