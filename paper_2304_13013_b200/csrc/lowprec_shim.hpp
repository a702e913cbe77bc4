// lowprec_shim.hpp — the reference's `lowprec::` operator API (proj/core/include/lowprec/
// {matrix,quantize,linear,optimizer}.hpp) served by the B200 C-ABI (include/switchback_b200.h).
//
// Same names, signatures, value semantics and std::invalid_argument messages as the reference,
// so its call sites (model.cpp, bench.cpp, noise.cpp, trainer.cpp) and its unit tests relink
// unchanged (option A). Host `Matrix` in, host `Matrix` out; every numeric op
// runs on the B200 in the reference-bit-exact mode (fp32 I/O, fp64 dequant epilogue, sequential
// fp32 GEMMs). Pure data generators / scalar helpers (Rng, gaussian_matrix, derive_seed,
// finite_difference_grad, fp8_value_set, fp8_cast_scalar, beta2_warmup) are host code as in the
// reference — they are not on the path.
#pragma once

#include <cstdint>
#include <functional>
#include <initializer_list>
#include <random>
#include <string>
#include <utility>
#include <vector>

namespace lowprec {

// ------------------------------------------------------------------ matrix.hpp
class Matrix {
 public:
  Matrix() = default;
  Matrix(int64_t rows, int64_t cols, float fill = 0.0f);
  static Matrix from(std::initializer_list<std::initializer_list<float>> rows);
  int64_t rows() const { return r_; }
  int64_t cols() const { return c_; }
  int64_t size() const { return r_ * c_; }
  bool empty() const { return r_ == 0 || c_ == 0; }
  bool same_shape(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_; }
  float& operator()(int64_t i, int64_t j) { return v_[static_cast<size_t>(i * c_ + j)]; }
  const float& operator()(int64_t i, int64_t j) const { return v_[static_cast<size_t>(i * c_ + j)]; }
  float* data() { return v_.data(); }
  const float* data() const { return v_.data(); }
  bool all_finite() const;
  float abs_max() const;
  Matrix transposed() const;

 private:
  int64_t r_ = 0, c_ = 0;
  std::vector<float> v_;
};

bool operator==(const Matrix& a, const Matrix& b);
inline bool operator!=(const Matrix& a, const Matrix& b) { return !(a == b); }

Matrix matmul(const Matrix& a, const Matrix& b_transposed);  // B200: sequential fp32 kernel

class Rng {
 public:
  explicit Rng(uint64_t seed) : e_(seed) {}
  uint64_t next_u64() { return e_(); }
  double uniform01() { return double(e_() >> 11) * 0x1.0p-53; }
  double gaussian();
  float gaussian(float mean, float stdev) { return float(double(mean) + double(stdev) * gaussian()); }
  int64_t uniform_int(int64_t n) { return int64_t(e_() % uint64_t(n)); }

 private:
  std::mt19937_64 e_;
};

uint64_t derive_seed(uint64_t seed, uint64_t stream);
Matrix gaussian_matrix(int64_t rows, int64_t cols, float mean, float stdev, uint64_t seed);
Matrix finite_difference_grad(const std::function<double(const Matrix&)>& f, const Matrix& x, double step);

// ---------------------------------------------------------------- quantize.hpp
enum class QuantAxis { kRow, kColumn, kTensor };

struct Fp8Format {
  enum class Reserved { kTopExponent, kTopEncodingOnly };
  int exponent_bits = 4;
  int mantissa_bits = 3;
  int exponent_bias = 7;
  Reserved reserved = Reserved::kTopEncodingOnly;
  static Fp8Format e4m3() { return {4, 3, 7, Reserved::kTopEncodingOnly}; }
  static Fp8Format e5m2() { return {5, 2, 15, Reserved::kTopExponent}; }
  double max_finite() const;
};
bool operator==(const Fp8Format& a, const Fp8Format& b);

std::vector<float> fp8_value_set(const Fp8Format& fmt);
Matrix fp8_cast(const Matrix& x, const Fp8Format& fmt);
float fp8_cast_scalar(float x, const std::vector<float>& sorted_values);

struct QuantizedMatrix {
  int64_t rows = 0;
  int64_t cols = 0;
  QuantAxis axis = QuantAxis::kTensor;
  bool fp8 = false;
  std::vector<int8_t> payload_int8;
  std::vector<float> payload_fp8;
  std::vector<float> state;
  int64_t size() const { return rows * cols; }
  float state_for(int64_t i, int64_t j) const {
    return axis == QuantAxis::kRow ? state[size_t(i)] : axis == QuantAxis::kColumn ? state[size_t(j)] : state[0];
  }
};

QuantizedMatrix quantize_rowwise(const Matrix& x);
QuantizedMatrix quantize_columnwise(const Matrix& x);
QuantizedMatrix quantize_tensorwise(const Matrix& x);
QuantizedMatrix quantize_tensorwise_transpose(const Matrix& x);
QuantizedMatrix quantize_fp8(const Matrix& x, const Fp8Format& fmt, QuantAxis axis);
Matrix dequantize(const QuantizedMatrix& q);

// ------------------------------------------------------------------ linear.hpp
enum class LinearVariant { kStandard, kSwitchBack, kSwitchBackM, kSwitchBackQ, kAllQuant };
enum class NumericFormat { kInt8, kFp8 };
const char* to_string(LinearVariant v);
LinearVariant parse_linear_variant(const std::string& name);

struct LinearMode {
  LinearVariant variant = LinearVariant::kStandard;
  NumericFormat format = NumericFormat::kInt8;
  Fp8Format fp8_forward = Fp8Format::e4m3();
  Fp8Format fp8_gradient = Fp8Format::e5m2();
};
bool operator==(const LinearMode& a, const LinearMode& b);

struct LinearContext {
  LinearMode mode;
  Matrix x_full;
  Matrix w_full;
  QuantizedMatrix x_quant;
  QuantizedMatrix w_quant;
};

Matrix int8_matmul_dequant(const QuantizedMatrix& qx, const QuantizedMatrix& qw);
Matrix matmul_dequant_dual_rowwise(const QuantizedMatrix& qa, const QuantizedMatrix& qb);
Matrix linear_forward(const LinearMode& mode, const Matrix& x, const Matrix& w, LinearContext* ctx = nullptr);
std::pair<Matrix, Matrix> linear_backward(const LinearMode& mode, const LinearContext& ctx, const Matrix& g);

// --------------------------------------------------------------- optimizer.hpp
enum class Clipping { kNone, kUpdateClip, kGradClip };
const char* to_string(Clipping c);
Clipping parse_clipping(const std::string& name);

struct OptimizerHyperparams {
  std::function<double(int64_t)> lr_schedule;
  double beta1 = 0.9;
  double beta2 = 0.99;
  double beta2_warmup_lambda = 0.0;
  double eps = 1e-6;
  double weight_decay = 0.0;
  Clipping clipping = Clipping::kNone;
  double max_grad_norm = 1.0;
};

struct TensorOptState {
  Matrix v;
  Matrix u;
  static TensorOptState zeros(int64_t rows, int64_t cols);
};

struct LossScaler {
  double scale = 1.0;
  bool per_tensor_skip = true;
};

double compute_rms(const Matrix& g, const Matrix& u, double eps);
double beta2_warmup(int64_t t, double lambda);
void grad_clip_global_norm(std::vector<Matrix>& grads, double max_norm);

struct FilterResult {
  std::vector<Matrix> grads;
  std::vector<size_t> skipped;
};
FilterResult filter_nonfinite(const std::vector<Matrix>& grads, const LossScaler& scaler);

struct TensorStepInfo {
  double rms = 0.0;
  double eta = 0.0;
};

struct TensorRef {
  std::string name;
  Matrix* param = nullptr;
  const Matrix* grad = nullptr;
  TensorOptState* state = nullptr;
};

std::vector<TensorStepInfo> optimizer_step(std::vector<TensorRef>& tensors, const OptimizerHyperparams& hp, int64_t t);

}  // namespace lowprec
