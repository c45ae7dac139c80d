// dropin.cpp -- the reference C++ API (namespace dtq, include/dtq/*.hpp)
// implemented over the C ABI (include/dtq_capi.h) on the B200.
//
// Value semantics as in the reference: Matrix / QuantizedTensor hold host
// data; every quantize / dequantize / balance / qlinear call uploads its
// operands, runs the fp64 "exact" device kernels and downloads the result,
// so results are bit-identical to the reference library.  Error behaviour
// follows the reference: std::invalid_argument, std::overflow_error,
// std::logic_error; a CUDA failure (or no sm_100 device: there is no CPU
// fallback) raises std::runtime_error.
//
// Host-side pieces are bookkeeping and analysis only: grouping indices,
// round_even (the rounding definition), error_report / incoherence / mse, the
// calibration-time scaling mask and sign draw, byte accounting.  The
// calibration statistics (col_absmax / row_absmax), fwht and choose_alpha's
// matrices run on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>

#include "../../include/dtq/balance.hpp"
#include "../../include/dtq/matrix.hpp"
#include "../../include/dtq/plan.hpp"
#include "../../include/dtq/qgemm.hpp"
#include "../../include/dtq/quant.hpp"
#include "../../include/dtq_capi.h"

namespace dtq {
namespace {

void check(int status) {
  if (status == DTQ_OK) return;
  const std::string msg = dtq_last_error();
  switch (status) {
    case DTQ_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case DTQ_ERR_OVERFLOW: throw std::overflow_error(msg);
    case DTQ_ERR_UNSUPPORTED: throw std::logic_error(msg);
    default: throw std::runtime_error("dtq device error: " + msg);
  }
}

void cuda(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA: ") + cudaGetErrorString(e));
}

// Device buffers come from a per-thread pool of power-of-two blocks: the
// value-semantics API makes many small calls, and cudaMalloc / cudaFree per
// call would cost more than the kernels.
class DevicePool {
 public:
  void* get(std::size_t bytes) {
    const std::size_t b = bucket(bytes);
    auto it = free_.find(b);
    if (it != free_.end()) {
      void* p = it->second;
      free_.erase(it);
      return p;
    }
    void* p = nullptr;
    cuda(cudaMalloc(&p, b));
    return p;
  }
  void put(void* p, std::size_t bytes) {
    if (free_.size() < 256)
      free_.emplace(bucket(bytes), p);
    else
      cudaFree(p);
  }
  ~DevicePool() {
    for (auto& kv : free_) cudaFree(kv.second);
  }

 private:
  static std::size_t bucket(std::size_t n) {
    std::size_t b = 256;
    while (b < n) b <<= 1;
    return b;
  }
  std::multimap<std::size_t, void*> free_;
};

DevicePool& pool() {
  thread_local DevicePool p;
  return p;
}

// RAII device buffer
template <typename T>
struct Dev {
  T* p = nullptr;
  std::size_t n = 0;
  explicit Dev(std::size_t count) : n(count) {
    if (n) p = static_cast<T*>(pool().get(n * sizeof(T)));
  }
  Dev(const T* host, std::size_t count) : Dev(count) {
    if (n) cuda(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  ~Dev() {
    if (p) pool().put(p, n * sizeof(T));
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void get(T* host) const {
    if (n) cuda(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost));
  }
};

int grouping_code(Grouping g) { return static_cast<int>(g); }

int64_t pitch16(std::size_t cols) { return static_cast<int64_t>((cols + 15) / 16 * 16); }

// Dynamic params of `rows` contiguous groups of `cols` doubles (device).
void row_params(const double* x, std::size_t rows, std::size_t cols, int bits, bool symmetric,
                QuantParams* out) {
  if (rows == 0 || cols == 0) throw std::invalid_argument("quant: empty group");
  if (!bits_supported(bits)) throw std::invalid_argument("quant: bits must be one of {2,4,6,8}");
  Dev<double> dx(x, rows * cols);
  const int64_t ldc = pitch16(cols);
  Dev<uint8_t> dc(rows * ldc);
  Dev<double> ds(rows);
  Dev<int32_t> dz(rows), st(1);
  cuda(cudaMemset(st.p, 0, sizeof(int32_t)));
  check(dtq_quantize_rows(dx.p, DTQ_F64, rows, cols, cols, bits, symmetric ? 1 : 0, DTQ_MODE_EXACT,
                          nullptr, nullptr, dc.p, ldc, ds.p, dz.p, st.p, nullptr));
  int32_t bad = 0;
  st.get(&bad);
  if (bad) throw std::invalid_argument("quant: non-finite value in group");
  std::vector<double> s(rows);
  std::vector<int32_t> z(rows);
  ds.get(s.data());
  dz.get(z.data());
  for (std::size_t r = 0; r < rows; ++r) out[r] = {s[r], z[r], bits};
}

std::vector<double> transpose(const Matrix& m) {
  std::vector<double> t(m.size());
  for (std::size_t r = 0; r < m.rows(); ++r)
    for (std::size_t c = 0; c < m.cols(); ++c) t[c * m.rows() + r] = m(r, c);
  return t;
}

// codes for given per-group params (device, fp64 divide + half-even)
std::vector<uint8_t> codes_for(const Matrix& x, const GroupingScheme& scheme, int bits,
                               const std::vector<QuantParams>& params) {
  std::vector<double> s(params.size());
  std::vector<int32_t> z(params.size());
  for (std::size_t i = 0; i < params.size(); ++i) {
    s[i] = params[i].scale;
    z[i] = params[i].zero_point;
  }
  Dev<double> dx(x.data().data(), x.size()), ds(s.data(), s.size());
  Dev<int32_t> dz(z.data(), z.size());
  Dev<uint8_t> dc(x.size());
  check(dtq_quantize_static(dx.p, x.rows(), x.cols(), x.cols(), bits, grouping_code(scheme.kind),
                            scheme.group_size, ds.p, dz.p, dc.p, x.cols(), nullptr));
  std::vector<uint8_t> out(x.size());
  dc.get(out.data());
  return out;
}

// device QuantLinear handle built from the layer's host fields
// The device handle keeps per-handle scratch (codes, the s32 accumulator of
// the fp64 epilogue), so calls on one layer are serialised by its mutex: the
// reference API is thread-safe (pure functions on const layers) and stays so.
struct Handle {
  dtq_qlinear_t h = nullptr;
  uint64_t fingerprint = 0;  // of the host fields the handle was built from
  std::mutex m;
  ~Handle() {
    if (h) dtq_qlinear_destroy(h);
  }
};

std::mutex g_layer_mu;  // guards the lazy QuantLinear::device upload

// 64-bit hash of a byte range (8 bytes per step, multiply / xor-shift mixing)
uint64_t mix_bytes(uint64_t h, const void* data, std::size_t n) {
  const auto* p = static_cast<const unsigned char*>(data);
  auto mix = [](uint64_t v) {
    v ^= v >> 33;
    v *= 0xff51afd7ed558ccdULL;
    v ^= v >> 33;
    return v;
  };
  std::size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    uint64_t w;
    std::memcpy(&w, p + i, 8);
    h = mix(h ^ w) * 0x9e3779b97f4a7c15ULL;
  }
  uint64_t tail = 0;
  std::memcpy(&tail, p + i, n - i);
  return mix(h ^ tail ^ (static_cast<uint64_t>(n) << 56));
}

// The reference's qlinear_forward reads w_q, bias and act_bits on every call
// (qgemm.cpp:23-67): the device handle is keyed on all of them, so a layer
// whose fields change after its first forward (or a copy that diverges from
// the layer it was copied from) gets a fresh handle, never stale weights.
uint64_t layer_fingerprint(const QuantLinear& layer) {
  const QuantizedTensor& w = layer.w_q;
  uint64_t h = 0x243f6a8885a308d3ULL;
  const int64_t dims[4] = {static_cast<int64_t>(w.rows), static_cast<int64_t>(w.cols),
                           layer.act_bits, layer.bias ? static_cast<int64_t>(layer.bias->size()) : -1};
  h = mix_bytes(h, dims, sizeof(dims));
  h = mix_bytes(h, w.ints.data(), w.ints.size());
  for (const QuantParams& p : w.params) {
    h = mix_bytes(h, &p.scale, sizeof(p.scale));
    const int32_t zb[2] = {p.zero_point, p.bits};
    h = mix_bytes(h, zb, sizeof(zb));
  }
  if (layer.bias) h = mix_bytes(h, layer.bias->data(), layer.bias->size() * sizeof(double));
  return h;
}

std::shared_ptr<Handle> device_layer(const QuantLinear& layer) {
  const uint64_t fp = layer_fingerprint(layer);
  std::lock_guard<std::mutex> lock(g_layer_mu);
  if (layer.device) {
    auto cur = std::static_pointer_cast<Handle>(layer.device);
    if (cur->fingerprint == fp) return cur;
  }
  const QuantizedTensor& w = layer.w_q;
  if (w.params.size() != w.rows || w.ints.size() != w.rows * w.cols)
    throw std::invalid_argument("qlinear: malformed weight tensor");
  const int wbits = w.params.empty() ? 8 : w.params[0].bits;
  std::vector<double> s(w.rows);
  for (std::size_t o = 0; o < w.rows; ++o) {
    if (w.params[o].zero_point != (1 << (wbits - 1)))
      throw std::logic_error("qlinear: device GEMM expects symmetric weights (z = 2^(b-1))");
    s[o] = w.params[o].scale;
  }
  Dev<uint8_t> dc(w.ints.data(), w.ints.size());
  Dev<double> ds(s.data(), s.size());
  std::unique_ptr<Dev<double>> db;
  if (layer.bias) {
    if (layer.bias->size() != w.rows) throw std::invalid_argument("qlinear: bias length != C_out");
    db = std::make_unique<Dev<double>>(layer.bias->data(), layer.bias->size());
  }
  auto hd = std::make_shared<Handle>();
  check(dtq_qlinear_create_from_codes(dc.p, 0, w.cols, wbits, ds.p, w.rows, w.cols, layer.act_bits,
                                      db ? db->p : nullptr, nullptr, nullptr, &hd->h));
  cuda(cudaDeviceSynchronize());
  hd->fingerprint = fp;
  layer.device = hd;
  return hd;
}

Matrix balance_rows(const Matrix& m, const double* smooth, bool mul, const int8_t* signs,
                    std::size_t hb) {
  Dev<double> dx(m.data().data(), m.size()), dout(m.size());
  std::unique_ptr<Dev<double>> dsm;
  std::unique_ptr<Dev<int8_t>> dsg;
  if (smooth) dsm = std::make_unique<Dev<double>>(smooth, m.cols());
  if (signs) dsg = std::make_unique<Dev<int8_t>>(signs, m.cols());
  check(dtq_balance_apply(dx.p, m.rows(), m.cols(), m.cols(), dsm ? dsm->p : nullptr, mul ? 1 : 0,
                          dsg ? dsg->p : nullptr, hb, dout.p, m.cols(), nullptr));
  Matrix out(m.rows(), m.cols());
  dout.get(out.data().data());
  return out;
}

}  // namespace

// ================================================================ matrix.hpp
Matrix matmul_nt(const Matrix& x, const Matrix& w) {
  if (x.cols() != w.cols()) throw std::invalid_argument("matmul_nt: inner dimensions differ");
  Dev<double> dx(x.data().data(), x.size()), dw(w.data().data(), w.size());
  Dev<double> dy(x.rows() * w.rows());
  check(dtq_matmul_nt_f64(dx.p, x.rows(), x.cols(), dw.p, w.rows(), nullptr, dy.p, nullptr));
  Matrix y(x.rows(), w.rows());
  dy.get(y.data().data());
  return y;
}

double max_abs(const Matrix& m) {
  double v = 0.0;
  for (double x : m.data()) v = std::max(v, std::abs(x));
  return v;
}

double mse(const Matrix& a, const Matrix& b) {
  if (!a.same_shape(b)) throw std::invalid_argument("mse: shape mismatch");
  double acc = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) acc += (a.data()[i] - b.data()[i]) * (a.data()[i] - b.data()[i]);
  return acc / static_cast<double>(a.size());
}

// calibration statistics on the device (max is exact: any reduction order
// gives the reference's values)
std::vector<double> col_absmax(const Matrix& m) {
  std::vector<double> out(m.cols(), 0.0);
  if (m.rows() == 0 || m.cols() == 0) return out;
  Dev<double> dx(m.data().data(), m.size()), dout(m.cols());
  check(dtq_col_absmax_f64(dx.p, m.rows(), m.cols(), m.cols(), dout.p, nullptr));
  dout.get(out.data());
  return out;
}

std::vector<double> row_absmax(const Matrix& m) {
  std::vector<double> out(m.rows(), 0.0);
  if (m.rows() == 0 || m.cols() == 0) return out;
  Dev<double> dx(m.data().data(), m.size()), dout(m.rows());
  check(dtq_row_absmax_f64(dx.p, m.rows(), m.cols(), m.cols(), dout.p, nullptr));
  dout.get(out.data());
  return out;
}

// ================================================================ quant.hpp
double round_even(double v) {
  // IEEE roundToIntegralTiesToEven (quant.cpp:9-16 restates it with floor/fmod)
  return std::nearbyint(v);
}

bool bits_supported(int bits) { return bits == 2 || bits == 4 || bits == 6 || bits == 8; }

std::size_t GroupingScheme::group_count(std::size_t rows, std::size_t cols) const {
  switch (kind) {
    case Grouping::PerTensor: return 1;
    case Grouping::PerToken:
    case Grouping::PerOutputChannel: return rows;
    case Grouping::PerChannel: return cols;
    case Grouping::PerGroup:
      if (group_size == 0 || cols % group_size != 0)
        throw std::invalid_argument("GroupingScheme: group_size must divide cols");
      return rows * (cols / group_size);
  }
  throw std::logic_error("GroupingScheme: bad kind");
}

std::size_t GroupingScheme::group_of(std::size_t r, std::size_t c, std::size_t cols) const {
  switch (kind) {
    case Grouping::PerTensor: return 0;
    case Grouping::PerToken:
    case Grouping::PerOutputChannel: return r;
    case Grouping::PerChannel: return c;
    case Grouping::PerGroup: return r * (cols / group_size) + c / group_size;
  }
  throw std::logic_error("GroupingScheme: bad kind");
}

QuantParams compute_minmax_params(std::span<const double> group, int bits) {
  QuantParams p;
  row_params(group.data(), group.empty() ? 0 : 1, group.size(), bits, false, &p);
  return p;
}

QuantParams compute_symmetric_params(std::span<const double> group, int bits) {
  QuantParams p;
  row_params(group.data(), group.empty() ? 0 : 1, group.size(), bits, true, &p);
  return p;
}

std::vector<QuantParams> compute_params(const Matrix& x, const GroupingScheme& scheme, int bits,
                                        bool symmetric) {
  const std::size_t ng = scheme.group_count(x.rows(), x.cols());
  std::vector<QuantParams> p(ng);
  switch (scheme.kind) {
    case Grouping::PerToken:
    case Grouping::PerOutputChannel:
      row_params(x.data().data(), x.rows(), x.cols(), bits, symmetric, p.data());
      break;
    case Grouping::PerGroup:  // contiguous sub-rows: rows * (cols/gs) groups of gs
      row_params(x.data().data(), ng, scheme.group_size, bits, symmetric, p.data());
      break;
    case Grouping::PerTensor:
      row_params(x.data().data(), 1, x.size(), bits, symmetric, p.data());
      break;
    case Grouping::PerChannel: {
      const std::vector<double> t = transpose(x);
      row_params(t.data(), x.cols(), x.rows(), bits, symmetric, p.data());
      break;
    }
  }
  return p;
}

QuantizedTensor quantize(const Matrix& x, const GroupingScheme& scheme, int bits, QuantMode mode,
                         const std::vector<QuantParams>* frozen_params, bool symmetric) {
  if (!bits_supported(bits)) throw std::invalid_argument("quantize: bits must be one of {2,4,6,8}");
  if (!x.all_finite()) throw std::invalid_argument("quantize: non-finite input");
  const std::size_t ng = scheme.group_count(x.rows(), x.cols());
  QuantizedTensor q;
  q.rows = x.rows();
  q.cols = x.cols();
  q.scheme = scheme;
  q.symmetric = symmetric;
  if (mode == QuantMode::Static) {
    if (frozen_params == nullptr)
      throw std::invalid_argument("quantize: Static mode requires frozen params");
    if (frozen_params->size() != ng)
      throw std::invalid_argument("quantize: frozen params group count mismatch");
    for (const auto& p : *frozen_params)
      if (p.bits != bits) throw std::invalid_argument("quantize: frozen params bit width mismatch");
    q.params = *frozen_params;
  } else {
    q.params = compute_params(x, scheme, bits, symmetric);
  }
  q.ints = codes_for(x, scheme, bits, q.params);
  return q;
}

Matrix dequantize(const QuantizedTensor& q) {
  Matrix out(q.rows, q.cols);
  std::vector<double> s(q.params.size());
  std::vector<int32_t> z(q.params.size());
  for (std::size_t i = 0; i < q.params.size(); ++i) {
    s[i] = q.params[i].scale;
    z[i] = q.params[i].zero_point;
  }
  Dev<uint8_t> dc(q.ints.data(), q.ints.size());
  Dev<double> ds(s.data(), s.size()), dout(out.size());
  Dev<int32_t> dz(z.data(), z.size());
  check(dtq_dequantize(dc.p, q.rows, q.cols, q.cols, grouping_code(q.scheme.kind),
                       q.scheme.group_size, ds.p, dz.p, dout.p, q.cols, nullptr));
  dout.get(out.data().data());
  return out;
}

Matrix fake_quantize(const Matrix& x, const GroupingScheme& scheme, int bits, QuantMode mode,
                     const std::vector<QuantParams>* frozen_params, bool symmetric) {
  return dequantize(quantize(x, scheme, bits, mode, frozen_params, symmetric));
}

QuantErrorReport error_report(const Matrix& x, const QuantizedTensor& q) {
  if (x.rows() != q.rows || x.cols() != q.cols)
    throw std::invalid_argument("error_report: shape mismatch");
  QuantErrorReport rep;
  double rnd = 0.0, clp = 0.0;
  for (std::size_t r = 0; r < q.rows; ++r)
    for (std::size_t c = 0; c < q.cols; ++c) {
      const QuantParams& p = q.params_of(r, c);
      const double pre = round_even(x(r, c) / p.scale) + p.zero_point;
      const double err = x(r, c) - p.scale * (static_cast<int32_t>(q.code(r, c)) - p.zero_point);
      rep.max_abs_err = std::max(rep.max_abs_err, std::abs(err));
      ((pre < 0.0 || pre > static_cast<double>((1 << p.bits) - 1)) ? clp : rnd) += err * err;
    }
  const double n = static_cast<double>(x.size());
  rep.rounding_mse = rnd / n;
  rep.clamping_mse = clp / n;
  rep.total_mse = (rnd + clp) / n;
  return rep;
}

double incoherence(std::span<const double> group) {
  if (group.empty()) throw std::invalid_argument("incoherence: empty group");
  double amax = 0.0, sq = 0.0;
  for (double v : group) {
    amax = std::max(amax, std::abs(v));
    sq += v * v;
  }
  if (sq == 0.0) throw std::invalid_argument("incoherence: all-zero group");
  return amax * std::sqrt(static_cast<double>(group.size())) / std::sqrt(sq);
}

// ================================================================ balance.hpp
void fwht(double* data, std::size_t n) {
  // on the device, the reference's butterfly order (balance.cpp:22-33); the
  // reference's loop reads past the end for n that is not a power of two
  if (n <= 1) return;
  if ((n & (n - 1)) != 0) throw std::invalid_argument("fwht: n must be a power of two");
  Dev<double> dx(data, n);
  check(dtq_fwht_f64(dx.p, 1, static_cast<int64_t>(n), static_cast<int64_t>(n), nullptr));
  dx.get(data);
}

ScalingMask compute_scaling_mask(const std::vector<double>& act_absmax,
                                 const std::vector<double>& weight_absmax, double alpha) {
  if (act_absmax.size() != weight_absmax.size())
    throw std::invalid_argument("compute_scaling_mask: vector length mismatch");
  if (alpha < 0.0 || alpha > 1.0)
    throw std::invalid_argument("compute_scaling_mask: alpha must be in [0,1]");
  ScalingMask m;
  m.alpha = alpha;
  m.s.resize(act_absmax.size());
  for (std::size_t i = 0; i < act_absmax.size(); ++i) {
    const double a = act_absmax[i], w = weight_absmax[i];
    const bool dead = a <= 0.0 || w <= 0.0 || !std::isfinite(a) || !std::isfinite(w);
    m.s[i] = dead ? 1.0 : std::clamp(std::pow(a, alpha) / std::pow(w, 1.0 - alpha), 1e-5, 1e5);
  }
  return m;
}

std::pair<Matrix, Matrix> apply_scaling(const Matrix& x, const Matrix& w, const ScalingMask& mask) {
  if (x.cols() != mask.s.size() || w.cols() != mask.s.size())
    throw std::invalid_argument("apply_scaling: dimension mismatch");
  return {balance_rows(x, mask.s.data(), false, nullptr, 0),
          balance_rows(w, mask.s.data(), true, nullptr, 0)};
}

RotationMatrix hadamard_matrix(std::size_t n, bool randomize, uint64_t seed) {
  if (n < 2 || (n & (n - 1)) != 0)
    throw std::invalid_argument("hadamard_matrix: n must be a power of two >= 2");
  RotationMatrix h;
  h.n = n;
  h.sign_diag.assign(n, int8_t{1});
  if (randomize) {
    std::mt19937_64 rng(seed);
    for (auto& d : h.sign_diag) d = (rng() & 1) ? int8_t{1} : int8_t{-1};
  }
  return h;
}

Matrix RotationMatrix::dense() const {
  Matrix m(n, n);
  const double norm = 1.0 / std::sqrt(static_cast<double>(n));
  for (std::size_t r = 0; r < n; ++r)
    for (std::size_t c = 0; c < n; ++c)
      m(r, c) = sign_diag[r] * ((std::popcount(r & c) & 1) ? -1 : 1) * norm;
  return m;
}

Matrix rotate_channels(const Matrix& m, const RotationMatrix& h) {
  if (m.cols() != h.n) throw std::invalid_argument("rotate_channels: channel count != rotation size");
  return balance_rows(m, nullptr, false, h.sign_diag.data(), h.n);
}

std::pair<Matrix, Matrix> apply_rotation(const Matrix& x, const Matrix& w, const RotationMatrix& h) {
  if (x.cols() != h.n || w.cols() != h.n)
    throw std::invalid_argument("apply_rotation: dimension mismatch");
  return {rotate_channels(x, h), rotate_channels(w, h)};
}

BalanceTransform static_dynamic_balance(const Matrix& static_base, const Matrix& w, double alpha,
                                        uint64_t seed) {
  if (static_base.cols() != w.cols())
    throw std::invalid_argument("static_dynamic_balance: channel mismatch");
  BalanceTransform t;
  t.mask = compute_scaling_mask(col_absmax(static_base), col_absmax(w), alpha);
  t.rotation = hadamard_matrix(w.cols(), true, seed);
  return t;
}

std::pair<Matrix, Matrix> apply_balance(const Matrix& x, const Matrix& w, const BalanceTransform& t) {
  Matrix xb = x, wb = w;
  if (t.mask) std::tie(xb, wb) = apply_scaling(xb, wb, *t.mask);
  if (t.rotation) std::tie(xb, wb) = apply_rotation(xb, wb, *t.rotation);
  return {std::move(xb), std::move(wb)};
}

namespace {

// fake_quantize(v, per-row group, bits, Dynamic, symmetric) in place on the
// device: exact per-row params and codes (quant.cpp:90-177), then
// dequantize (quant.cpp:179-188) over the same buffer
void fake_quantize_rows_dev(double* v, std::size_t rows, std::size_t cols, int bits,
                            bool symmetric, int grouping) {
  const int64_t ldc = pitch16(cols);
  Dev<uint8_t> dc(rows * ldc);
  Dev<double> ds(rows);
  Dev<int32_t> dz(rows), st(1);
  cuda(cudaMemset(st.p, 0, sizeof(int32_t)));
  check(dtq_quantize_rows(v, DTQ_F64, rows, cols, cols, bits, symmetric ? 1 : 0, DTQ_MODE_EXACT,
                          nullptr, nullptr, dc.p, ldc, ds.p, dz.p, st.p, nullptr));
  int32_t bad = 0;
  st.get(&bad);
  if (bad) throw std::invalid_argument("quantize: non-finite input");
  check(dtq_dequantize(dc.p, rows, cols, ldc, grouping, 0, ds.p, dz.p, v, cols, nullptr));
}

}  // namespace

// choose_alpha (balance.cpp:142-165) with every matrix resident on the
// device: the reference GEMM, the column statistics, both sides of
// apply_scaling, the per-token / per-output-channel fake quantization and the
// quantized GEMM of each alpha.  The mask (K pow() per alpha) and the mse
// (the reference's sequential fp64 sum, which sets the ordering of nearly
// equal errors) stay on the host, so the chosen alpha is the reference's.
double choose_alpha(const Matrix& calib_x, const Matrix& w, int act_bits, int weight_bits) {
  if (calib_x.cols() != w.cols()) throw std::invalid_argument("matmul_nt: inner dimensions differ");
  const std::size_t M = calib_x.rows(), K = calib_x.cols(), N = w.rows();
  if (M == 0 || K == 0 || N == 0) throw std::invalid_argument("choose_alpha: empty input");
  if (!bits_supported(act_bits) || !bits_supported(weight_bits))
    throw std::invalid_argument("quantize: bits must be one of {2,4,6,8}");
  Dev<double> dx(calib_x.data().data(), M * K), dw(w.data().data(), N * K);
  Dev<double> dy(M * N), dxs(M * K), dws(N * K), dam(K), dwm(K), dsm(K);
  check(dtq_matmul_nt_f64(dx.p, M, K, dw.p, N, nullptr, dy.p, nullptr));
  Matrix ref(M, N);
  dy.get(ref.data().data());
  std::vector<double> am(K), wm(K);
  check(dtq_col_absmax_f64(dx.p, M, K, K, dam.p, nullptr));
  check(dtq_col_absmax_f64(dw.p, N, K, K, dwm.p, nullptr));
  dam.get(am.data());
  dwm.get(wm.data());
  double best_alpha = 0.5, best = std::numeric_limits<double>::infinity();
  Matrix yq(M, N);
  for (int step = 1; step <= 9; ++step) {
    const double alpha = 0.1 * step;
    const ScalingMask mask = compute_scaling_mask(am, wm, alpha);
    cuda(cudaMemcpy(dsm.p, mask.s.data(), K * sizeof(double), cudaMemcpyHostToDevice));
    check(dtq_balance_apply(dx.p, M, K, K, dsm.p, 0, nullptr, 0, dxs.p, K, nullptr));  // X / s
    check(dtq_balance_apply(dw.p, N, K, K, dsm.p, 1, nullptr, 0, dws.p, K, nullptr));  // W * s
    fake_quantize_rows_dev(dxs.p, M, K, act_bits, false, 1);      // per_token, asymmetric
    fake_quantize_rows_dev(dws.p, N, K, weight_bits, true, 3);    // per_output_channel, symmetric
    check(dtq_matmul_nt_f64(dxs.p, M, K, dws.p, N, nullptr, dy.p, nullptr));
    dy.get(yq.data().data());
    const double err = mse(yq, ref);
    if (err < best) {
      best = err;
      best_alpha = alpha;
    }
  }
  return best_alpha;
}

// ================================================================ qgemm.hpp
QuantLinear make_quant_linear(const Matrix& w, int weight_bits, int act_bits,
                              const std::optional<std::vector<double>>& bias) {
  if (!bits_supported(weight_bits) || !bits_supported(act_bits))
    throw std::invalid_argument("make_quant_linear: unsupported bit width");
  if (bias && bias->size() != w.rows())
    throw std::invalid_argument("make_quant_linear: bias length != C_out");
  if (!w.all_finite()) throw std::invalid_argument("quantize: non-finite input");
  Dev<double> dw(w.data().data(), w.size());
  std::unique_ptr<Dev<double>> db;
  if (bias) db = std::make_unique<Dev<double>>(bias->data(), bias->size());
  auto hd = std::make_shared<Handle>();
  check(dtq_qlinear_create(dw.p, DTQ_F64, w.rows(), w.cols(), w.cols(), weight_bits, act_bits,
                           db ? db->p : nullptr, nullptr, nullptr, &hd->h));
  QuantLinear layer;
  layer.w_q.rows = w.rows();
  layer.w_q.cols = w.cols();
  layer.w_q.scheme = GroupingScheme::per_output_channel();
  layer.w_q.symmetric = true;
  layer.w_q.ints.resize(w.size());
  std::vector<double> s(w.rows());
  check(dtq_qlinear_export(hd->h, layer.w_q.ints.data(), s.data(), nullptr, nullptr));
  layer.w_q.params.resize(w.rows());
  for (std::size_t o = 0; o < w.rows(); ++o) layer.w_q.params[o] = {s[o], 1 << (weight_bits - 1), weight_bits};
  layer.bias = bias;
  layer.act_bits = act_bits;
  hd->fingerprint = layer_fingerprint(layer);
  layer.device = hd;
  return layer;
}

Matrix qlinear_forward(const Matrix& x, const QuantLinear& layer) {
  const std::size_t c_in = layer.in_channels(), c_out = layer.out_channels();
  if (x.cols() != c_in) throw std::invalid_argument("qlinear_forward: X cols != C_in");
  const int64_t max_term =
      static_cast<int64_t>((1 << layer.act_bits) - 1) *
      (int64_t{1} << (layer.w_q.params.empty() ? 7 : layer.w_q.params[0].bits - 1));
  if (max_term > std::numeric_limits<int64_t>::max() / static_cast<int64_t>(c_in))
    throw std::overflow_error("qlinear_forward: accumulator could overflow");
  if (!x.all_finite()) throw std::invalid_argument("quantize: non-finite input");
  const std::shared_ptr<Handle> hd = device_layer(layer);
  Dev<double> dx(x.data().data(), x.size()), dy(x.rows() * c_out);
  Matrix y(x.rows(), c_out);
  {
    std::lock_guard<std::mutex> lock(hd->m);
    check(dtq_qlinear_forward(dx.p, DTQ_F64, x.rows(), c_in, hd->h, DTQ_MODE_EXACT, nullptr, dy.p,
                              DTQ_F64, c_out, nullptr, 0, nullptr, nullptr));
    dy.get(y.data().data());
  }
  return y;
}

Matrix qlinear_forward_float(const Matrix& x, const QuantLinear& layer) {
  const Matrix x_fq = fake_quantize(x, GroupingScheme::per_token(), layer.act_bits, QuantMode::Dynamic);
  const Matrix w_deq = dequantize(layer.w_q);
  Dev<double> dx(x_fq.data().data(), x_fq.size()), dw(w_deq.data().data(), w_deq.size());
  Dev<double> dy(x.rows() * w_deq.rows());
  std::unique_ptr<Dev<double>> db;
  if (layer.bias) db = std::make_unique<Dev<double>>(layer.bias->data(), layer.bias->size());
  check(dtq_matmul_nt_f64(dx.p, x_fq.rows(), x_fq.cols(), dw.p, w_deq.rows(), db ? db->p : nullptr,
                          dy.p, nullptr));
  Matrix y(x.rows(), w_deq.rows());
  dy.get(y.data().data());
  return y;
}

LayerBytes weight_bytes(std::size_t rows, std::size_t cols, int bits, std::size_t group_count) {
  return {(rows * cols * static_cast<std::size_t>(bits) + 7) / 8, group_count * 4};
}

std::size_t checkpoint_bytes(const std::vector<std::pair<Matrix, int>>& layers) {
  std::size_t total = 0;
  for (const auto& [w, bits] : layers) {
    const LayerBytes b = weight_bytes(w.rows(), w.cols(), bits, w.rows());
    total += b.weights + b.params;
  }
  return total;
}

std::size_t fp16_baseline_bytes(const std::vector<std::pair<Matrix, int>>& layers) {
  std::size_t total = 0;
  for (const auto& l : layers) total += l.first.rows() * l.first.cols() * 2;
  return total;
}

// ================================================================ plan.hpp
std::array<TimestepRange, kNumRanges> partition_timesteps(std::size_t steps) {
  if (steps == 0 || steps % kNumRanges != 0)
    throw std::invalid_argument("partition_timesteps: steps must be divisible by 4");
  std::array<TimestepRange, kNumRanges> out;
  const std::size_t span = steps / kNumRanges;
  for (std::size_t i = 0; i < kNumRanges; ++i) out[i] = {i, i * span, (i + 1) * span};
  return out;
}

}  // namespace dtq
