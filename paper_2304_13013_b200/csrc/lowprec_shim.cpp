// lowprec_shim.cpp — the reference's lowprec:: API (see lowprec_shim.hpp) on the B200 C-ABI.
//
// Each path function mirrors the reference's composition (linear.cpp:113-278,
// optimizer.cpp:102-172) but every numeric primitive — quantize, dequantize, int8 GEMM with the
// fp64 epilogue, the sequential fp32 matmul / weight gradient, fp8 snapping, StableAdamW, the
// RMS / clip / loss-scaler reductions, finiteness checks — is a kernel launched through
// include/switchback_b200.h. Host Matrix buffers are staged through device memory per call
// (the reference's value semantics: inputs const&, outputs by value).
#include "lowprec_shim.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "switchback_b200.h"

namespace lowprec {
namespace {

[[noreturn]] void raise(sb_status s) {
  const std::string msg = sb_last_error();
  if (s == SB_ERR_INVALID_ARGUMENT || s == SB_ERR_NONFINITE) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
void chk(sb_status s) {
  if (s != SB_OK) raise(s);
}

sb_handle H() {
  static sb_handle h = [] {
    sb_handle x = nullptr;
    const sb_status s = sb_create(0, &x);
    if (s != SB_OK) throw std::runtime_error(std::string("lowprec_b200: ") + sb_last_error());
    return x;
  }();
  return h;
}

// Synchronize; a latched device-side non-finite flag becomes the reference's exception.
void sync_or_throw(const char* op) {
  const sb_status s = sb_synchronize(H());
  if (s == SB_ERR_NONFINITE) throw std::invalid_argument(std::string(op) + ": non-finite input");
  chk(s);
}

class Dev {
 public:
  Dev() = default;
  explicit Dev(size_t bytes) : n_(bytes) {
    if (bytes) chk(sb_device_alloc(H(), bytes, &p_));
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  Dev(Dev&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; }
  Dev& operator=(Dev&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  ~Dev() {
    if (p_) sb_device_free(H(), p_);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p_);
  }

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};

template <class T>
Dev up(const T* src, size_t count) {
  Dev d(count * sizeof(T));
  chk(sb_copy_to_device(H(), d.as<void>(), src, count * sizeof(T)));
  return d;
}
Dev up(const Matrix& m) { return up(m.data(), size_t(m.size())); }
template <class T>
void down(T* dst, const Dev& d, size_t count) {
  chk(sb_copy_to_host(H(), dst, d.as<void>(), count * sizeof(T)));
}
Matrix down_matrix(const Dev& d, int64_t r, int64_t c) {
  Matrix m(r, c);
  down(m.data(), d, size_t(r * c));
  return m;
}

sb_axis ax(QuantAxis a) {
  return a == QuantAxis::kRow ? SB_AXIS_ROW : a == QuantAxis::kColumn ? SB_AXIS_COLUMN : SB_AXIS_TENSOR;
}
size_t state_len(QuantAxis a, int64_t r, int64_t c) {
  return a == QuantAxis::kRow ? size_t(r) : a == QuantAxis::kColumn ? size_t(c) : 1;
}

int fp8_code(const Fp8Format& f, const char* op) {
  if (f == Fp8Format::e4m3()) return SB_E4M3;
  if (f == Fp8Format::e5m2()) return SB_E5M2;
  if (f.exponent_bits < 1 || f.mantissa_bits < 0 || f.exponent_bits + f.mantissa_bits != 7)
    throw std::invalid_argument("fp8: invalid bit split (need 1 sign + e + m == 8)");
  throw std::invalid_argument(std::string(op) + ": the B200 path implements e4m3 and e5m2");
}

void require_quantizable(const Matrix& x, const char* op) {  // quantize.cpp:11-14
  if (x.empty()) throw std::invalid_argument(std::string(op) + ": empty matrix");
}

QuantizedMatrix quantize_int8(const Matrix& x, QuantAxis axis, bool transposed, const char* op) {
  require_quantizable(x, op);
  const int64_t r = x.rows(), c = x.cols();
  Dev dx = up(x), dq(size_t(r * c)), ds(state_len(axis, r, c) * sizeof(float));
  sb_status s;
  if (axis == QuantAxis::kRow)
    s = sb_quantize_rowwise(H(), dx.as<void>(), SB_F32, r, c, c, dq.as<int8_t>(), c, ds.as<float>());
  else if (axis == QuantAxis::kColumn)
    s = sb_quantize_columnwise(H(), dx.as<void>(), SB_F32, r, c, c, dq.as<int8_t>(), c, nullptr, 0, ds.as<float>());
  else if (!transposed)
    s = sb_quantize_tensorwise(H(), dx.as<void>(), SB_F32, r, c, c, dq.as<int8_t>(), c, nullptr, 0, ds.as<float>());
  else
    s = sb_quantize_tensorwise(H(), dx.as<void>(), SB_F32, r, c, c, nullptr, 0, dq.as<int8_t>(), r, ds.as<float>());
  chk(s);
  sync_or_throw(op);
  QuantizedMatrix q;
  q.rows = transposed ? c : r;
  q.cols = transposed ? r : c;
  q.axis = axis;
  q.fp8 = false;
  q.payload_int8.resize(size_t(r * c));
  q.state.resize(state_len(axis, r, c));
  down(q.payload_int8.data(), dq, q.payload_int8.size());
  down(q.state.data(), ds, q.state.size());
  return q;
}

void check_finite(const Matrix& m) {
  if (m.size()) {
    Dev d = up(m);
    chk(sb_check_finite(H(), d.as<void>(), SB_F32, m.size()));
    chk(sb_synchronize(H()));
  }
}

// wgrad_full_precision (linear.cpp:193-195) == matmul(G^T, X^T): the device kernel sums the
// same products in the same (token) order without materialising the transposes.
Matrix wgrad(const Matrix& g, const Matrix& x) {
  const int64_t b = g.rows(), m = g.cols(), n = x.cols();
  Dev dg = up(g), dx = up(x), dw(size_t(m * n) * sizeof(float));
  chk(sb_wgrad(H(), dg.as<void>(), dx.as<void>(), SB_F32, b, m, n, dw.as<float>(), /*exact=*/1, 0));
  return down_matrix(dw, m, n);
}

// transpose_tensorwise, linear.cpp:170-189 (payload moved on the device)
QuantizedMatrix transpose_tensorwise(const QuantizedMatrix& q) {
  QuantizedMatrix t;
  t.rows = q.cols;
  t.cols = q.rows;
  t.axis = QuantAxis::kTensor;
  t.fp8 = q.fp8;
  t.state = q.state;
  if (q.fp8) {
    Matrix m(q.rows, q.cols);
    std::memcpy(m.data(), q.payload_fp8.data(), q.payload_fp8.size() * sizeof(float));
    Matrix mt = m.transposed();
    t.payload_fp8.assign(mt.data(), mt.data() + mt.size());
  } else {
    Dev in = up(q.payload_int8.data(), q.payload_int8.size()), out(q.payload_int8.size());
    chk(sb_transpose_i8(H(), in.as<int8_t>(), q.rows, q.cols, out.as<int8_t>()));
    t.payload_int8.resize(q.payload_int8.size());
    down(t.payload_int8.data(), out, t.payload_int8.size());
  }
  return t;
}

Matrix int8_product(const QuantizedMatrix& qa, const QuantizedMatrix& qb, sb_scale_mode mode) {  // linear.cpp:54-67
  if (qa.cols != qb.cols) throw std::invalid_argument("int8 matmul: inner dimension mismatch");
  const int64_t M = qa.rows, N = qb.rows, K = qa.cols;
  // the epilogue indexes A's state per row; a tensor-wise A is broadcast (linear.cpp:57-58)
  std::vector<float> sa(static_cast<size_t>(M)), sbv(mode == SB_SCALE_ROW_ROW ? size_t(N) : 1);
  for (int64_t i = 0; i < M; ++i) sa[size_t(i)] = qa.axis == QuantAxis::kRow ? qa.state[size_t(i)] : qa.state[0];
  if (mode == SB_SCALE_ROW_ROW)
    for (int64_t j = 0; j < N; ++j) sbv[size_t(j)] = qb.axis == QuantAxis::kRow ? qb.state[size_t(j)] : qb.state[0];
  else
    sbv[0] = qb.state[0];
  Dev a = up(qa.payload_int8.data(), qa.payload_int8.size()), b = up(qb.payload_int8.data(), qb.payload_int8.size());
  Dev dsa = up(sa.data(), sa.size()), dsb = up(sbv.data(), sbv.size()), y(size_t(M * N) * sizeof(float));
  if (M && N) chk(sb_gemm_i8(H(), a.as<int8_t>(), dsa.as<float>(), b.as<int8_t>(), dsb.as<float>(), mode, M, N, K,
                             y.as<void>(), SB_F32, /*exact=*/1));
  return down_matrix(y, M, N);
}

// fp8 simulation helpers (linear.cpp:164-178)
Matrix fp8_snap(const Matrix& m, const Fp8Format& fmt, QuantAxis axis) { return dequantize(quantize_fp8(m, fmt, axis)); }
QuantAxis fp8_weight_axis(LinearVariant v) { return v == LinearVariant::kSwitchBackQ ? QuantAxis::kRow : QuantAxis::kTensor; }
QuantAxis fp8_activation_axis(LinearVariant v) { return v == LinearVariant::kAllQuant ? QuantAxis::kTensor : QuantAxis::kRow; }

}  // namespace

// ================================================================ matrix.hpp
Matrix::Matrix(int64_t rows, int64_t cols, float fill) : r_(rows), c_(cols) {
  if (rows < 0 || cols < 0) throw std::invalid_argument("matrix: negative shape");
  v_.assign(size_t(rows) * size_t(cols), fill);
}

Matrix Matrix::from(std::initializer_list<std::initializer_list<float>> rows) {
  Matrix m(int64_t(rows.size()), rows.size() ? int64_t(rows.begin()->size()) : 0);
  int64_t i = 0;
  for (const auto& row : rows) {
    if (int64_t(row.size()) != m.c_) throw std::invalid_argument("matrix: ragged rows");
    std::copy(row.begin(), row.end(), m.v_.begin() + i * m.c_);
    ++i;
  }
  return m;
}

bool Matrix::all_finite() const {
  return std::all_of(v_.begin(), v_.end(), [](float v) { return std::isfinite(v); });
}

float Matrix::abs_max() const {
  float m = 0.0f;
  for (float v : v_) m = std::max(m, std::fabs(v));
  return m;
}

Matrix Matrix::transposed() const {
  Matrix t(c_, r_);
  for (int64_t i = 0; i < r_; ++i)
    for (int64_t j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
  return t;
}

bool operator==(const Matrix& a, const Matrix& b) {
  if (!a.same_shape(b)) return false;
  for (int64_t i = 0; i < a.size(); ++i)
    if (a.data()[i] != b.data()[i]) return false;
  return true;
}

Matrix matmul(const Matrix& a, const Matrix& bt) {  // matrix.cpp:53-68 on the device
  if (a.cols() != bt.cols()) throw std::invalid_argument("matmul: inner dimension mismatch");
  const int64_t r = a.rows(), c = bt.rows(), k = a.cols();
  Dev da = up(a), db = up(bt), dy(size_t(r * c) * sizeof(float));
  if (r && c) chk(sb_matmul_f32(H(), da.as<float>(), db.as<float>(), r, c, k, dy.as<float>()));
  return down_matrix(dy, r, c);
}

double Rng::gaussian() {  // Box-Muller on 53-bit uniforms (matrix.hpp:53-56)
  const double u1 = double((e_() >> 11) + 1) * 0x1.0p-53;
  const double u2 = double(e_() >> 11) * 0x1.0p-53;
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
}

uint64_t derive_seed(uint64_t seed, uint64_t stream) {  // splitmix64 finalizer
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

Matrix gaussian_matrix(int64_t rows, int64_t cols, float mean, float stdev, uint64_t seed) {
  if (stdev < 0) throw std::invalid_argument("gaussian_matrix: negative stdev");
  Matrix m(rows, cols);
  Rng rng(seed);
  for (int64_t i = 0; i < m.size(); ++i) m.data()[i] = rng.gaussian(mean, stdev);
  return m;
}

Matrix finite_difference_grad(const std::function<double(const Matrix&)>& f, const Matrix& x, double step) {
  if (step <= 0) throw std::invalid_argument("finite_difference_grad: step must be > 0");
  Matrix g(x.rows(), x.cols()), probe = x;
  for (int64_t i = 0; i < x.size(); ++i) {
    const float v = x.data()[i];
    const float hi = float(double(v) + step), lo = float(double(v) - step);
    probe.data()[i] = hi;
    const double fh = f(probe);
    probe.data()[i] = lo;
    const double fl = f(probe);
    probe.data()[i] = v;
    if (!std::isfinite(fh) || !std::isfinite(fl)) throw std::runtime_error("finite_difference_grad: non-finite evaluation");
    g.data()[i] = float((fh - fl) / (double(hi) - double(lo)));
  }
  return g;
}

// ============================================================== quantize.hpp
std::vector<float> fp8_value_set(const Fp8Format& fmt) {  // the format's definition
  if (fmt.exponent_bits < 1 || fmt.mantissa_bits < 0 || fmt.exponent_bits + fmt.mantissa_bits != 7)
    throw std::invalid_argument("fp8: invalid bit split (need 1 sign + e + m == 8)");
  const int emax = (1 << fmt.exponent_bits) - 1, mmax = (1 << fmt.mantissa_bits) - 1;
  std::vector<float> v;
  for (int e = 0; e <= emax; ++e)
    for (int m = 0; m <= mmax; ++m) {
      if (e == emax && (fmt.reserved == Fp8Format::Reserved::kTopExponent || m == mmax)) continue;
      const double val = e == 0 ? std::ldexp(double(m), 1 - fmt.exponent_bias - fmt.mantissa_bits)
                                : std::ldexp(1.0 + double(m) / double(1 << fmt.mantissa_bits), e - fmt.exponent_bias);
      v.push_back(float(val));
      v.push_back(float(-val));
    }
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  return v;
}

double Fp8Format::max_finite() const { return double(fp8_value_set(*this).back()); }

bool operator==(const Fp8Format& a, const Fp8Format& b) {
  return a.exponent_bits == b.exponent_bits && a.mantissa_bits == b.mantissa_bits &&
         a.exponent_bias == b.exponent_bias && a.reserved == b.reserved;
}

float fp8_cast_scalar(float x, const std::vector<float>& v) {  // scalar helper over a caller-given set
  auto it = std::lower_bound(v.begin(), v.end(), x);
  if (it == v.end()) return v.back();
  if (it == v.begin() || *it == x) return *it;
  const float hi = *it, lo = *(it - 1);
  const double dh = double(hi) - double(x), dl = double(x) - double(lo);
  if (dl < dh) return lo;
  if (dh < dl) return hi;
  return std::fabs(lo) <= std::fabs(hi) ? lo : hi;
}

Matrix fp8_cast(const Matrix& x, const Fp8Format& fmt) {
  const int code = fp8_code(fmt, "fp8_cast");
  Dev dx = up(x), dy(size_t(x.size()) * sizeof(float));
  chk(sb_fp8_cast(H(), dx.as<float>(), x.size(), sb_fp8_format(code), dy.as<float>()));
  sync_or_throw("fp8_cast");
  return down_matrix(dy, x.rows(), x.cols());
}

QuantizedMatrix quantize_rowwise(const Matrix& x) { return quantize_int8(x, QuantAxis::kRow, false, "quantize_rowwise"); }
QuantizedMatrix quantize_columnwise(const Matrix& x) {
  return quantize_int8(x, QuantAxis::kColumn, false, "quantize_columnwise");
}
QuantizedMatrix quantize_tensorwise(const Matrix& x) {
  return quantize_int8(x, QuantAxis::kTensor, false, "quantize_tensorwise");
}
QuantizedMatrix quantize_tensorwise_transpose(const Matrix& x) {
  return quantize_int8(x, QuantAxis::kTensor, true, "quantize_tensorwise_transpose");
}

QuantizedMatrix quantize_fp8(const Matrix& x, const Fp8Format& fmt, QuantAxis axis) {
  const int code = fp8_code(fmt, "quantize_fp8");
  require_quantizable(x, "quantize_fp8");
  const int64_t r = x.rows(), c = x.cols();
  const size_t ns = state_len(axis, r, c);
  Dev dx = up(x), dq(size_t(r * c)), ds(ns * sizeof(float)), dv(size_t(r * c) * sizeof(float));
  chk(sb_quantize_fp8(H(), dx.as<void>(), SB_F32, r, c, c, sb_fp8_format(code), ax(axis), dq.as<uint8_t>(), c,
                      ds.as<float>()));
  sync_or_throw("quantize_fp8");
  // decoded payload values (the reference stores fp8 payloads as their fp32 values)
  const float one = 1.0f;
  Dev d1 = up(&one, 1);
  chk(sb_dequantize_fp8(H(), dq.as<uint8_t>(), r, c, c, sb_fp8_format(code), d1.as<float>(), SB_AXIS_TENSOR,
                        dv.as<void>(), SB_F32, c));
  QuantizedMatrix q;
  q.rows = r;
  q.cols = c;
  q.axis = axis;
  q.fp8 = true;
  q.payload_fp8.resize(size_t(r * c));
  q.state.resize(ns);
  down(q.payload_fp8.data(), dv, q.payload_fp8.size());
  down(q.state.data(), ds, ns);
  return q;
}

Matrix dequantize(const QuantizedMatrix& q) {
  if (q.state.size() != state_len(q.axis, q.rows, q.cols))
    throw std::invalid_argument("dequantize: state length does not match axis");
  Dev ds = up(q.state.data(), q.state.size()), dy(size_t(q.size()) * sizeof(float));
  if (q.size() == 0) return Matrix(q.rows, q.cols);
  if (q.fp8) {
    Dev dp = up(q.payload_fp8.data(), q.payload_fp8.size());
    chk(sb_dequantize_values(H(), dp.as<float>(), q.rows, q.cols, ds.as<float>(), ax(q.axis), dy.as<float>()));
  } else {
    Dev dp = up(q.payload_int8.data(), q.payload_int8.size());
    chk(sb_dequantize(H(), dp.as<int8_t>(), q.rows, q.cols, q.cols, ds.as<float>(), ax(q.axis), dy.as<void>(), SB_F32,
                      q.cols));
  }
  return down_matrix(dy, q.rows, q.cols);
}

// ================================================================ linear.hpp
const char* to_string(LinearVariant v) {
  switch (v) {
    case LinearVariant::kStandard: return "Standard";
    case LinearVariant::kSwitchBack: return "SwitchBack";
    case LinearVariant::kSwitchBackM: return "SwitchBackM";
    case LinearVariant::kSwitchBackQ: return "SwitchBackQ";
    case LinearVariant::kAllQuant: return "AllQuant";
  }
  return "?";
}

LinearVariant parse_linear_variant(const std::string& name) {
  for (LinearVariant v : {LinearVariant::kStandard, LinearVariant::kSwitchBack, LinearVariant::kSwitchBackM,
                          LinearVariant::kSwitchBackQ, LinearVariant::kAllQuant})
    if (name == to_string(v)) return v;
  throw std::invalid_argument("unknown linear variant: " + name);
}

bool operator==(const LinearMode& a, const LinearMode& b) {
  if (a.variant != b.variant || a.format != b.format) return false;
  if (a.format == NumericFormat::kInt8) return true;
  return a.fp8_forward == b.fp8_forward && a.fp8_gradient == b.fp8_gradient;
}

Matrix int8_matmul_dequant(const QuantizedMatrix& qx, const QuantizedMatrix& qw) {
  if (qx.fp8 || qw.fp8) throw std::invalid_argument("int8_matmul_dequant: fp8 operand");
  if (qx.axis != QuantAxis::kRow || qw.axis != QuantAxis::kTensor)
    throw std::invalid_argument("int8_matmul_dequant: need row-wise X and tensor-wise W");
  return int8_product(qx, qw, SB_SCALE_ROW_TENSOR);
}

Matrix matmul_dequant_dual_rowwise(const QuantizedMatrix& qa, const QuantizedMatrix& qb) {
  if (qa.fp8 || qb.fp8) throw std::invalid_argument("matmul_dequant_dual_rowwise: fp8 operand");
  if (qa.axis != QuantAxis::kRow || qb.axis != QuantAxis::kRow)
    throw std::invalid_argument("matmul_dequant_dual_rowwise: both operands must be row-wise");
  return int8_product(qa, qb, SB_SCALE_ROW_ROW);
}

Matrix linear_forward(const LinearMode& mode, const Matrix& x, const Matrix& w, LinearContext* ctx) {
  // check_forward_shapes, linear.cpp:87-93
  if (x.empty() || w.empty()) throw std::invalid_argument("linear_forward: empty operand");
  if (x.cols() != w.cols()) throw std::invalid_argument("linear_forward: X is b x n but W is not m x n");
  try {
    check_finite(x);
    check_finite(w);
  } catch (const std::invalid_argument&) {
    throw std::invalid_argument("linear_forward: non-finite input");
  }
  if (ctx) {
    *ctx = LinearContext{};
    ctx->mode = mode;
  }
  if (mode.variant == LinearVariant::kStandard) {
    if (ctx) {
      ctx->x_full = x;
      ctx->w_full = w;
    }
    return matmul(x, w);
  }
  if (mode.format == NumericFormat::kInt8) {
    Matrix y = mode.variant == LinearVariant::kSwitchBackQ
                   ? matmul_dequant_dual_rowwise(quantize_rowwise(x), quantize_rowwise(w))
                   : int8_matmul_dequant(quantize_rowwise(x), quantize_tensorwise(w));
    if (ctx) {
      if (mode.variant == LinearVariant::kSwitchBackM) {
        ctx->x_quant = quantize_rowwise(x);
        ctx->w_quant = quantize_tensorwise(w);
      } else {
        ctx->x_full = x;
        ctx->w_full = w;
      }
    }
    return y;
  }
  QuantizedMatrix qx = quantize_fp8(x, mode.fp8_forward, fp8_activation_axis(mode.variant));
  QuantizedMatrix qw = quantize_fp8(w, mode.fp8_forward, fp8_weight_axis(mode.variant));
  Matrix y = matmul(dequantize(qx), dequantize(qw));
  if (ctx) {
    if (mode.variant == LinearVariant::kSwitchBackM) {
      ctx->x_quant = std::move(qx);
      ctx->w_quant = std::move(qw);
    } else {
      ctx->x_full = x;
      ctx->w_full = w;
    }
  }
  return y;
}

std::pair<Matrix, Matrix> linear_backward(const LinearMode& mode, const LinearContext& ctx, const Matrix& g) {
  if (!(mode == ctx.mode)) throw std::invalid_argument("linear_backward: context was produced by a different mode");
  const bool qs = ctx.mode.variant == LinearVariant::kSwitchBackM;
  const int64_t b = qs ? ctx.x_quant.rows : ctx.x_full.rows();
  const int64_t m = qs ? ctx.w_quant.rows : ctx.w_full.rows();
  if (g.rows() != b || g.cols() != m) throw std::invalid_argument("linear_backward: G must be b x m");

  if (mode.variant == LinearVariant::kStandard)
    return {matmul(g, ctx.w_full.transposed()), wgrad(g, ctx.x_full)};

  if (mode.format == NumericFormat::kInt8) {
    Matrix x_grad;
    if (mode.variant == LinearVariant::kSwitchBackQ)
      x_grad = matmul_dequant_dual_rowwise(quantize_rowwise(g), quantize_rowwise(ctx.w_full.transposed()));
    else if (mode.variant == LinearVariant::kSwitchBackM)
      x_grad = int8_matmul_dequant(quantize_rowwise(g), transpose_tensorwise(ctx.w_quant));
    else
      x_grad = int8_matmul_dequant(quantize_rowwise(g), quantize_tensorwise_transpose(ctx.w_full));
    Matrix w_grad;
    if (mode.variant == LinearVariant::kAllQuant)
      w_grad = matmul_dequant_dual_rowwise(quantize_rowwise(g.transposed()), quantize_rowwise(ctx.x_full.transposed()));
    else if (mode.variant == LinearVariant::kSwitchBackM)
      w_grad = wgrad(g, dequantize(ctx.x_quant));
    else
      w_grad = wgrad(g, ctx.x_full);
    return {std::move(x_grad), std::move(w_grad)};
  }

  Matrix w_snap_t;
  if (mode.variant == LinearVariant::kSwitchBackM)
    w_snap_t = dequantize(ctx.w_quant).transposed();
  else if (mode.variant == LinearVariant::kSwitchBackQ)
    w_snap_t = dequantize(quantize_fp8(ctx.w_full.transposed(), mode.fp8_forward, QuantAxis::kRow));
  else
    w_snap_t = dequantize(quantize_fp8(ctx.w_full, mode.fp8_forward, fp8_weight_axis(mode.variant))).transposed();
  const QuantAxis gx = mode.variant == LinearVariant::kAllQuant ? QuantAxis::kTensor : QuantAxis::kRow;
  Matrix g_snap = fp8_snap(g, mode.fp8_gradient, gx);
  Matrix x_grad = matmul(g_snap, w_snap_t);
  Matrix w_grad;
  if (mode.variant == LinearVariant::kAllQuant)
    w_grad = wgrad(g_snap, fp8_snap(ctx.x_full, mode.fp8_forward, QuantAxis::kTensor));
  else if (mode.variant == LinearVariant::kSwitchBackM)
    w_grad = wgrad(g, dequantize(ctx.x_quant));
  else
    w_grad = wgrad(g, ctx.x_full);
  return {std::move(x_grad), std::move(w_grad)};
}

// ============================================================= optimizer.hpp
const char* to_string(Clipping c) {
  switch (c) {
    case Clipping::kNone: return "none";
    case Clipping::kUpdateClip: return "update_clip";
    case Clipping::kGradClip: return "grad_clip";
  }
  return "?";
}

Clipping parse_clipping(const std::string& name) {
  if (name == "none") return Clipping::kNone;
  if (name == "update_clip") return Clipping::kUpdateClip;
  if (name == "grad_clip") return Clipping::kGradClip;
  throw std::invalid_argument("unknown clipping mode: " + name);
}

TensorOptState TensorOptState::zeros(int64_t rows, int64_t cols) {
  TensorOptState s;
  s.v = Matrix(rows, cols);
  s.u = Matrix(rows, cols);
  return s;
}

double compute_rms(const Matrix& g, const Matrix& u, double eps) {
  if (!g.same_shape(u)) throw std::invalid_argument("compute_rms: shape mismatch");
  Dev dg = up(g), du = up(u), out(sizeof(double));
  chk(sb_compute_rms(H(), dg.as<float>(), du.as<float>(), g.size(), eps, out.as<double>()));
  double r = 0.0;
  down(&r, out, 1);
  return r;
}

double beta2_warmup(int64_t t, double lambda) {  // optimizer.cpp:44-49 (scalar schedule)
  if (t < 1) throw std::invalid_argument("beta2_warmup: t must be >= 1");
  if (lambda <= 0) throw std::invalid_argument("beta2_warmup: lambda must be > 0");
  return std::min(1.0 - std::pow(double(t), -lambda), std::nextafter(1.0, 0.0));
}

void grad_clip_global_norm(std::vector<Matrix>& grads, double max_norm) {
  if (max_norm <= 0) throw std::invalid_argument("grad_clip: max_norm must be > 0");
  std::vector<Dev> d;
  std::vector<float*> ptrs;
  std::vector<int64_t> numel;
  for (const Matrix& g : grads) {
    d.push_back(up(g));
    ptrs.push_back(d.back().as<float>());
    numel.push_back(g.size());
  }
  chk(sb_grad_clip_global_norm(H(), ptrs.data(), numel.data(), int(grads.size()), max_norm));
  for (size_t i = 0; i < grads.size(); ++i) down(grads[i].data(), d[i], size_t(grads[i].size()));
}

FilterResult filter_nonfinite(const std::vector<Matrix>& grads, const LossScaler& scaler) {
  if (!(scaler.scale > 0)) throw std::invalid_argument("loss scaler: scale must be > 0");
  FilterResult r;
  const int n = int(grads.size());
  std::vector<Dev> din, dout;
  std::vector<const float*> pin;
  std::vector<float*> pout;
  std::vector<int64_t> numel;
  for (const Matrix& g : grads) {
    din.push_back(up(g));
    dout.emplace_back(size_t(g.size()) * sizeof(float));
    pin.push_back(din.back().as<float>());
    pout.push_back(dout.back().as<float>());
    numel.push_back(g.size());
  }
  Dev flags(sizeof(int32_t) * size_t(std::max(n, 1)));
  chk(sb_filter_nonfinite(H(), pin.data(), pout.data(), numel.data(), n, scaler.scale, scaler.per_tensor_skip ? 1 : 0,
                          flags.as<int32_t>()));
  std::vector<int32_t> f(size_t(std::max(n, 1)));
  down(f.data(), flags, size_t(n));
  for (int i = 0; i < n; ++i) {
    r.grads.push_back(down_matrix(dout[size_t(i)], grads[size_t(i)].rows(), grads[size_t(i)].cols()));
    if (f[size_t(i)]) r.skipped.push_back(size_t(i));
  }
  return r;
}

std::vector<TensorStepInfo> optimizer_step(std::vector<TensorRef>& tensors, const OptimizerHyperparams& hp, int64_t t) {
  if (t < 1) throw std::invalid_argument("optimizer_step: t must be >= 1");
  if (!hp.lr_schedule) throw std::invalid_argument("optimizer_step: lr_schedule not set");
  for (const TensorRef& ref : tensors) {
    if (!ref.param || !ref.grad || !ref.state) throw std::invalid_argument("optimizer_step: null tensor reference");
    if (!ref.param->same_shape(*ref.grad) || !ref.param->same_shape(ref.state->v) ||
        !ref.param->same_shape(ref.state->u))
      throw std::invalid_argument("optimizer_step: shape mismatch for " + ref.name);
  }
  const int n = int(tensors.size());
  std::vector<Dev> bufs;
  std::vector<sb_adamw_tensor> desc(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    TensorRef& r = tensors[size_t(i)];
    bufs.push_back(up(*r.param));
    bufs.push_back(up(*r.grad));
    bufs.push_back(up(r.state->v));
    bufs.push_back(up(r.state->u));
    desc[size_t(i)] = sb_adamw_tensor{bufs[bufs.size() - 4].as<float>(), bufs[bufs.size() - 3].as<float>(),
                                      bufs[bufs.size() - 2].as<float>(), bufs[bufs.size() - 1].as<float>(),
                                      r.param->size()};
  }
  sb_adamw_hparams h{hp.lr_schedule(t), hp.beta1, hp.beta2, hp.beta2_warmup_lambda, hp.eps, hp.weight_decay,
                     hp.max_grad_norm, int32_t(hp.clipping)};
  size_t ws_bytes = 0;
  chk(sb_stableadamw_workspace_size(desc.data(), n, &ws_bytes));
  Dev ws(ws_bytes), rms(sizeof(double) * size_t(std::max(n, 1))), eta(sizeof(double) * size_t(std::max(n, 1)));
  chk(sb_stableadamw_step(H(), desc.data(), n, &h, t, rms.as<double>(), eta.as<double>(), ws.as<void>(), ws_bytes));
  std::vector<double> hr(size_t(std::max(n, 1))), he(size_t(std::max(n, 1)));
  down(hr.data(), rms, size_t(n));
  down(he.data(), eta, size_t(n));
  std::vector<TensorStepInfo> infos(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    TensorRef& r = tensors[size_t(i)];
    down(r.param->data(), bufs[size_t(4 * i)], size_t(r.param->size()));
    down(r.state->v.data(), bufs[size_t(4 * i + 2)], size_t(r.param->size()));
    down(r.state->u.data(), bufs[size_t(4 * i + 3)], size_t(r.param->size()));
    infos[size_t(i)] = TensorStepInfo{hr[size_t(i)], he[size_t(i)]};
  }
  return infos;
}

}  // namespace lowprec
