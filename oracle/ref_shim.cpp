// ref_shim.cpp -- C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference sources under /root/reference/proj/core/src (never copied into
// this repo) into oracle/_ref/libdtq_ref.so.  Used to pin the C restatement
// (dtq_oracle.c), to generate tests/golden fixtures, and as the CPU arm of
// bench.py (`--impl reference`, `cpu_baseline.kind = "reference"`).
//
// Each entry point calls the reference's own public API (dtq::quantize,
// dtq::make_quant_linear, dtq::qlinear_forward, dtq::rotate_channels,
// dtq::hadamard_matrix, dtq::compute_scaling_mask, dtq::apply_scaling,
// dtq::pack_codes/unpack_codes) and converts
// exceptions to status codes: 1 invalid_argument, 2 overflow_error, 4 other.

#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <stdexcept>
#include <thread>
#include <vector>

#include "dtq/balance.hpp"
#include "dtq/matrix.hpp"
#include "dtq/qgemm.hpp"
#include "dtq/quant.hpp"
#include "dtq/trace_io.hpp"

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::overflow_error&) {
    return 2;
  } catch (...) {
    return 4;
  }
}

dtq::Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
  return dtq::Matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
                     std::vector<double>(p, p + rows * cols));
}

dtq::QuantLinear make_layer(const uint8_t* wc, const double* sw, const int32_t* zw,
                            int wbits, int64_t N, int64_t K, const double* bias,
                            int act_bits) {
  dtq::QuantLinear layer;
  layer.w_q.rows = static_cast<std::size_t>(N);
  layer.w_q.cols = static_cast<std::size_t>(K);
  layer.w_q.ints.assign(wc, wc + N * K);
  layer.w_q.scheme = dtq::GroupingScheme::per_output_channel();
  layer.w_q.symmetric = true;
  layer.w_q.params.resize(static_cast<std::size_t>(N));
  for (int64_t o = 0; o < N; ++o) layer.w_q.params[o] = {sw[o], zw[o], wbits};
  if (bias) layer.bias = std::vector<double>(bias, bias + N);
  layer.act_bits = act_bits;
  return layer;
}

}  // namespace

extern "C" {

int dtq_ref_quantize_rows(const double* x, int64_t rows, int64_t cols, int bits,
                          int symmetric, uint8_t* codes, double* s, int32_t* z) {
  return guarded([&] {
    const dtq::Matrix m = to_matrix(x, rows, cols);
    const auto scheme = symmetric ? dtq::GroupingScheme::per_output_channel()
                                  : dtq::GroupingScheme::per_token();
    const dtq::QuantizedTensor q =
        dtq::quantize(m, scheme, bits, dtq::QuantMode::Dynamic, nullptr, symmetric != 0);
    std::memcpy(codes, q.ints.data(), q.ints.size());
    for (int64_t r = 0; r < rows; ++r) {
      s[r] = q.params[r].scale;
      z[r] = q.params[r].zero_point;
    }
  });
}

int dtq_ref_minmax_params(const double* g, int64_t n, int bits, double* s, int32_t* z) {
  return guarded([&] {
    const dtq::QuantParams p =
        dtq::compute_minmax_params(std::span<const double>(g, static_cast<std::size_t>(n)), bits);
    *s = p.scale;
    *z = p.zero_point;
  });
}

int dtq_ref_make_quant_linear(const double* w, int64_t N, int64_t K, int wbits, int act_bits,
                              uint8_t* codes, double* sw, int32_t* zw) {
  return guarded([&] {
    const dtq::QuantLinear layer = dtq::make_quant_linear(to_matrix(w, N, K), wbits, act_bits);
    std::memcpy(codes, layer.w_q.ints.data(), layer.w_q.ints.size());
    for (int64_t o = 0; o < N; ++o) {
      sw[o] = layer.w_q.params[o].scale;
      zw[o] = layer.w_q.params[o].zero_point;
    }
  });
}

// dtq::qlinear_forward over row slices on `threads` std::threads (SPEC.md:257
// permits row-parallel execution; per-token quantization is row-local, so the
// output is bit-identical to one whole-matrix call).  threads <= 1 is the
// reference exactly as shipped.
int dtq_ref_qlinear_forward(const double* x, int64_t M, int64_t K, const uint8_t* wc,
                            const double* sw, const int32_t* zw, int wbits, int64_t N,
                            const double* bias, int act_bits, double* y, int threads) {
  return guarded([&] {
    const dtq::QuantLinear layer = make_layer(wc, sw, zw, wbits, N, K, bias, act_bits);
    if (threads <= 1 || M < 2) {
      const dtq::Matrix out = dtq::qlinear_forward(to_matrix(x, M, K), layer);
      std::memcpy(y, out.data().data(), sizeof(double) * static_cast<std::size_t>(M * N));
      return;
    }
    const int64_t T = std::min<int64_t>(threads, M);
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(T));
    for (int64_t t = 0; t < T; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int64_t r0 = M * t / T, r1 = M * (t + 1) / T;
          if (r1 <= r0) return;
          const dtq::Matrix out =
              dtq::qlinear_forward(to_matrix(x + r0 * K, r1 - r0, K), layer);
          std::memcpy(y + r0 * N, out.data().data(),
                      sizeof(double) * static_cast<std::size_t>((r1 - r0) * N));
        } catch (...) {
          errs[static_cast<std::size_t>(t)] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

int dtq_ref_qlinear_forward_float(const double* x, int64_t M, int64_t K, const uint8_t* wc,
                                  const double* sw, const int32_t* zw, int wbits, int64_t N,
                                  const double* bias, int act_bits, double* y) {
  return guarded([&] {
    const dtq::QuantLinear layer = make_layer(wc, sw, zw, wbits, N, K, bias, act_bits);
    const dtq::Matrix out = dtq::qlinear_forward_float(to_matrix(x, M, K), layer);
    std::memcpy(y, out.data().data(), sizeof(double) * static_cast<std::size_t>(M * N));
  });
}

int dtq_ref_hadamard_signs(int64_t n, int randomize, uint64_t seed, int8_t* out) {
  return guarded([&] {
    const dtq::RotationMatrix h =
        dtq::hadamard_matrix(static_cast<std::size_t>(n), randomize != 0, seed);
    std::memcpy(out, h.sign_diag.data(), static_cast<std::size_t>(n));
  });
}

// reference rotate_channels applied per hblock-wide column block (hblock ==
// cols is the reference call itself).
int dtq_ref_rotate_blocks(double* x, int64_t rows, int64_t cols, int64_t hblock,
                          const int8_t* signs) {
  return guarded([&] {
    if (hblock <= 0 || cols % hblock != 0) throw std::invalid_argument("hblock");
    for (int64_t j = 0; j < cols; j += hblock) {
      dtq::Matrix blk(static_cast<std::size_t>(rows), static_cast<std::size_t>(hblock));
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < hblock; ++c) blk(r, c) = x[r * cols + j + c];
      dtq::RotationMatrix h;
      h.n = static_cast<std::size_t>(hblock);
      h.sign_diag.assign(signs + j, signs + j + hblock);
      const dtq::Matrix out = dtq::rotate_channels(blk, h);
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < hblock; ++c) x[r * cols + j + c] = out(r, c);
    }
  });
}

int dtq_ref_scaling_mask(const double* act_amax, const double* w_amax, int64_t n,
                         double alpha, double* s_out) {
  return guarded([&] {
    const dtq::ScalingMask m = dtq::compute_scaling_mask(
        std::vector<double>(act_amax, act_amax + n), std::vector<double>(w_amax, w_amax + n),
        alpha);
    std::memcpy(s_out, m.s.data(), sizeof(double) * static_cast<std::size_t>(n));
  });
}

int dtq_ref_apply_scaling(double* x, int64_t M, double* w, int64_t N, int64_t K,
                          const double* s) {
  return guarded([&] {
    dtq::ScalingMask m;
    m.s.assign(s, s + K);
    auto [xs, ws] = dtq::apply_scaling(to_matrix(x, M, K), to_matrix(w, N, K), m);
    std::memcpy(x, xs.data().data(), sizeof(double) * static_cast<std::size_t>(M * K));
    std::memcpy(w, ws.data().data(), sizeof(double) * static_cast<std::size_t>(N * K));
  });
}

double dtq_ref_round_even(double v) { return dtq::round_even(v); }

// trace_io.cpp:79-109 (the W4 nibble layout the W4A8 loader consumes)
int64_t dtq_ref_pack_codes(const uint8_t* codes, int64_t count, int bits, uint8_t* out) {
  int64_t n = -1;
  const int st = guarded([&] {
    const std::vector<uint8_t> p =
        dtq::pack_codes(std::span<const uint8_t>(codes, static_cast<std::size_t>(count)), bits);
    std::memcpy(out, p.data(), p.size());
    n = static_cast<int64_t>(p.size());
  });
  return st ? -1 : n;
}

// trace_io.cpp:225-261: write a checkpoint of n layers, each quantized by the
// reference's make_quant_linear path (quantize, per-output-channel,
// symmetric) at bits[i]; mask[i] (length K[i] or 0) and rot[i] (+-1, length
// K[i] or 0) are stored as given.  Used to generate tests/golden fixtures.
int dtq_ref_write_checkpoint(const char* path, int n, const char* const* names,
                             const double* const* w, const int64_t* N, const int64_t* K,
                             const int* bits, const float* const* mask,
                             const int8_t* const* rot) {
  return guarded([&] {
    dtq::QuantCheckpoint ck;
    for (int i = 0; i < n; ++i) {
      dtq::CheckpointLayer layer;
      layer.name = names[i];
      layer.weights = dtq::quantize(to_matrix(w[i], N[i], K[i]),
                                    dtq::GroupingScheme::per_output_channel(), bits[i],
                                    dtq::QuantMode::Dynamic, nullptr, /*symmetric=*/true);
      if (mask[i]) layer.mask.assign(mask[i], mask[i] + K[i]);
      if (rot[i]) layer.rotation_diag.assign(rot[i], rot[i] + K[i]);
      ck.layers.push_back(std::move(layer));
    }
    dtq::write_checkpoint(path, ck);
  });
}

// trace_io.cpp:263-316: read layer i back -- unpacked codes [N*K], the
// per-row scales as read (f32 widened to f64) and the zero points.
int dtq_ref_read_checkpoint_layer(const char* path, int64_t i, uint8_t* codes, double* scale,
                                  int32_t* zero, int64_t* n_layers) {
  return guarded([&] {
    const dtq::QuantCheckpoint ck = dtq::read_checkpoint(path);
    *n_layers = static_cast<int64_t>(ck.layers.size());
    const auto& w = ck.layers.at(static_cast<std::size_t>(i)).weights;
    std::memcpy(codes, w.ints.data(), w.ints.size());
    for (std::size_t o = 0; o < w.params.size(); ++o) {
      scale[o] = w.params[o].scale;
      zero[o] = w.params[o].zero_point;
    }
  });
}

}  // extern "C"
