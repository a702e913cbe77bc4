/*
 * oracle.c — CPU restatement of the lowprec SwitchBack hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the B200
 * kernels: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference arm may load it. The product path never calls it (there is no CPU
 * fallback anywhere in paper_2304_13013_b200/).
 *
 * Every function restates the reference algorithm in plain C and cites the
 * reference file:line it follows (paths relative to /root/reference/proj/core).
 * Compiled with -O2 -ffp-contract=off, mirroring the reference's global
 * no-FMA contract (proj/CMakeLists.txt:12-17).
 *
 * Parity is pinned two ways (see tests/test_oracle_golden.py):
 *   - the known-answer vectors of proj/tests/{quantize,linear,optimizer,matrix}_test.cpp,
 *   - golden fixtures produced by the reference itself (oracle/_ref, built by
 *     oracle/Makefile from the reference sources), committed under tests/golden/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EMPTY 1
#define ORC_NONFINITE 2
#define ORC_BADARG 3

enum { ORC_ROW = 0, ORC_COL = 1, ORC_TENSOR = 2 };

/* ---------------------------------------------------------------- RNG ---- */
/* std::mt19937_64 (matrix.hpp:57-72), restated from the published MT19937-64
 * recurrence (Matsumoto & Nishimura 2000; parameters fixed by [rand.predef]). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

static void mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(orc_mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
    }
    s->idx = 0;
  }
  uint64_t y = s->mt[s->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* Rng::gaussian, matrix.cpp:70-75: Box-Muller on two 53-bit uniforms. */
static double mt64_gaussian(orc_mt64* s) {
  double u1 = (double)((mt64_next(s) >> 11) + 1) * 0x1.0p-53;
  double u2 = (double)(mt64_next(s) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* derive_seed, matrix.cpp:77-83 (splitmix64 finalizer). */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* gaussian_matrix, matrix.cpp:85-92 (row-major fill, Rng::gaussian(mean, stdev)
 * of matrix.hpp:64-66). */
int orc_gaussian_matrix(int64_t rows, int64_t cols, float mean, float stdev, uint64_t seed,
                        float* out) {
  if (stdev < 0) return ORC_BADARG;
  orc_mt64 s;
  mt64_seed(&s, seed);
  for (int64_t i = 0; i < rows * cols; ++i)
    out[i] = (float)((double)mean + (double)stdev * mt64_gaussian(&s));
  return ORC_OK;
}

/* Rng::uniform_int, matrix.hpp:68 — exposed so tests can rebuild the
 * reference fixtures (integer_grid, grid_matrix). */
void orc_uniform_int_stream(uint64_t seed, int64_t n, int64_t count, int64_t* out) {
  orc_mt64 s;
  mt64_seed(&s, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)(mt64_next(&s) % (uint64_t)n);
}

/* ----------------------------------------------------------- quantize ---- */
static int all_finite(const float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}

/* quantize_entry, quantize.cpp:17-20: lround(127*x/absmax) clamped to ±127. */
static int8_t quantize_entry(float x, float absmax) {
  long v = lround(127.0 * (double)x / (double)absmax);
  if (v < -127) v = -127;
  if (v > 127) v = 127;
  return (int8_t)v;
}

/* slice_absmax, quantize.cpp:89-112 (+ Matrix::abs_max, matrix.cpp:32-36):
 * exact max of |x| per slice; an all-zero slice gets the sentinel state 1.0. */
static void slice_absmax(const float* x, int64_t rows, int64_t cols, int axis, float* state) {
  int64_t ns = axis == ORC_ROW ? rows : axis == ORC_COL ? cols : 1;
  for (int64_t s = 0; s < ns; ++s) state[s] = 0.0f;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      int64_t s = axis == ORC_ROW ? i : axis == ORC_COL ? j : 0;
      float a = fabsf(x[i * cols + j]);
      if (a > state[s]) state[s] = a;
    }
  for (int64_t s = 0; s < ns; ++s)
    if (state[s] == 0.0f) state[s] = 1.0f;
}

/* quantize_int8, quantize.cpp:116-129 (row: :131-133, column: :135-137,
 * tensor: :139-141). require_quantizable (:11-14) -> ORC_EMPTY / ORC_NONFINITE. */
int orc_quantize_int8(const float* x, int64_t rows, int64_t cols, int axis, int8_t* q,
                      float* state) {
  if (rows == 0 || cols == 0) return ORC_EMPTY;
  if (!all_finite(x, rows * cols)) return ORC_NONFINITE;
  slice_absmax(x, rows, cols, axis, state);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      float s = axis == ORC_ROW ? state[i] : axis == ORC_COL ? state[j] : state[0];
      q[i * cols + j] = quantize_entry(x[i * cols + j], s);
    }
  return ORC_OK;
}

/* quantize_tensorwise_transpose, quantize.cpp:143-159: payload written at the
 * transposed position (cols x rows). */
int orc_quantize_tensorwise_transpose(const float* x, int64_t rows, int64_t cols, int8_t* qt,
                                      float* state) {
  if (rows == 0 || cols == 0) return ORC_EMPTY;
  if (!all_finite(x, rows * cols)) return ORC_NONFINITE;
  slice_absmax(x, rows, cols, ORC_TENSOR, state);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) qt[j * rows + i] = quantize_entry(x[i * cols + j], state[0]);
  return ORC_OK;
}

/* dequantize int8 branch, quantize.cpp:178-184,191-195. */
void orc_dequantize_int8(const int8_t* q, const float* state, int axis, int64_t rows, int64_t cols,
                         float* y) {
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      float s = axis == ORC_ROW ? state[i] : axis == ORC_COL ? state[j] : state[0];
      y[i * cols + j] = (float)((double)q[i * cols + j] * (double)s / 127.0);
    }
}

/* -------------------------------------------------------------- fp8 ------ */
/* fp8_value_set, quantize.cpp:30-56. reserved: 0 = top exponent reserved
 * (E5M2 convention), 1 = only the top encoding is NaN (E4M3 convention). */
static int cmp_float(const void* a, const void* b) {
  float x = *(const float*)a, y = *(const float*)b;
  return x < y ? -1 : x > y ? 1 : 0;
}

int orc_fp8_value_set(int ebits, int mbits, int bias, int reserved_top_exponent, float* out) {
  if (ebits < 1 || mbits < 0 || ebits + mbits != 7) return -1;
  int emax = (1 << ebits) - 1, mmax = (1 << mbits) - 1, n = 0;
  for (int e = 0; e <= emax; ++e)
    for (int m = 0; m <= mmax; ++m) {
      if (e == emax) {
        if (reserved_top_exponent) continue;
        if (m == mmax) continue;
      }
      double v = e == 0 ? ldexp((double)m, 1 - bias - mbits)
                        : ldexp(1.0 + (double)m / (double)(1 << mbits), e - bias);
      out[n++] = (float)v;
      out[n++] = (float)(-v);
    }
  qsort(out, (size_t)n, sizeof(float), cmp_float);
  int w = 0; /* std::unique: drops the duplicate zero */
  for (int r = 0; r < n; ++r)
    if (w == 0 || out[r] != out[w - 1]) out[w++] = out[r];
  return w;
}

/* fp8_cast_scalar, quantize.cpp:65-76: lower_bound, nearest, ties to the
 * smaller magnitude, saturate at the set edges. */
float orc_fp8_cast_scalar(float x, const float* v, int n) {
  int lo = 0, hi = n; /* first index with v[idx] >= x */
  while (lo < hi) {
    int mid = (lo + hi) / 2;
    if (v[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  if (lo == n) return v[n - 1];
  if (lo == 0 || v[lo] == x) return v[lo];
  float h = v[lo], l = v[lo - 1];
  double dh = (double)h - (double)x, dl = (double)x - (double)l;
  if (dl < dh) return l;
  if (dh < dl) return h;
  return fabsf(l) <= fabsf(h) ? l : h;
}

/* quantize_fp8, quantize.cpp:161-176: payload = snap(f32(x/state)). */
int orc_quantize_fp8(const float* x, int64_t rows, int64_t cols, int ebits, int mbits, int bias,
                     int reserved_top_exponent, int axis, float* payload, float* state) {
  if (rows == 0 || cols == 0) return ORC_EMPTY;
  if (!all_finite(x, rows * cols)) return ORC_NONFINITE;
  float vs[256];
  int n = orc_fp8_value_set(ebits, mbits, bias, reserved_top_exponent, vs);
  if (n < 0) return ORC_BADARG;
  slice_absmax(x, rows, cols, axis, state);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      float s = axis == ORC_ROW ? state[i] : axis == ORC_COL ? state[j] : state[0];
      payload[i * cols + j] = orc_fp8_cast_scalar((float)((double)x[i * cols + j] / (double)s), vs, n);
    }
  return ORC_OK;
}

/* ------------------------------------------------------------ GEMMs ------ */
/* accumulate_int8 / int8_product, linear.cpp:37-67: acc_ij = sum_k qa_ik*qb_jk
 * (int32 while k <= INT32_MAX/16129 = 133144, int64 beyond — the integer sum is
 * the same either way), y_ij = f32(double(acc)*sa_i*sb_j/16129).
 * sa/sb hold one state per row of qa/qb (a tensor-wise operand passes its single
 * state broadcast with sa_stride/sb_stride = 0). raw (nullable) receives acc. */
void orc_int8_gemm(const int8_t* qa, const float* sa, int64_t sa_stride, const int8_t* qb,
                   const float* sb, int64_t sb_stride, int64_t r, int64_t c, int64_t k,
                   int64_t* raw, float* y) {
  for (int64_t i = 0; i < r; ++i) {
    const int8_t* ai = qa + i * k;
    for (int64_t j = 0; j < c; ++j) {
      const int8_t* bj = qb + j * k;
      int64_t acc = 0;
      for (int64_t p = 0; p < k; ++p) acc += (int64_t)ai[p] * (int64_t)bj[p];
      if (raw) raw[i * c + j] = acc;
      if (y)
        y[i * c + j] = (float)((double)acc * (double)sa[i * sa_stride] * (double)sb[j * sb_stride] /
                               16129.0);
    }
  }
}

/* matmul, matrix.cpp:53-68: A (r x k) times B^T with B given as (c x k);
 * strictly sequential fp32 reduction per output (no FMA: -ffp-contract=off). */
void orc_matmul_f32(const float* a, const float* bt, int64_t r, int64_t c, int64_t k, float* y) {
  for (int64_t i = 0; i < r; ++i)
    for (int64_t j = 0; j < c; ++j) {
      const float* ai = a + i * k;
      const float* bj = bt + j * k;
      float acc = 0.0f;
      for (int64_t p = 0; p < k; ++p) acc += ai[p] * bj[p];
      y[i * c + j] = acc;
    }
}

/* wgrad_full_precision, linear.cpp:193-195: dW = matmul(G^T, X^T), i.e.
 * dW_ij = sum over tokens t (sequential, in order) of G_ti * X_tj.
 * G is b x m, X is b x n, dW is m x n. */
void orc_wgrad_f32(const float* g, const float* x, int64_t b, int64_t m, int64_t n, float* dw) {
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      float acc = 0.0f;
      for (int64_t t = 0; t < b; ++t) acc += g[t * m + i] * x[t * n + j];
      dw[i * n + j] = acc;
    }
}

/* ------------------------------------------------------- SwitchBack ------ */
/* linear_forward {kSwitchBack, kInt8}, linear.cpp:113-146 (int8 branch :128-146):
 * Y = int8_matmul_dequant(quantize_rowwise(X), quantize_tensorwise(W)).
 * X b x n, W m x n, Y b x m. Scratch-free: allocates its own payloads. */
int orc_switchback_forward(const float* x, const float* w, int64_t b, int64_t n, int64_t m,
                           float* y) {
  if (b == 0 || n == 0 || m == 0) return ORC_EMPTY; /* check_forward_shapes :87-93 */
  if (!all_finite(x, b * n) || !all_finite(w, m * n)) return ORC_NONFINITE;
  int8_t* qx = (int8_t*)malloc((size_t)(b * n));
  int8_t* qw = (int8_t*)malloc((size_t)(m * n));
  float* sx = (float*)malloc((size_t)b * sizeof(float));
  float sw;
  orc_quantize_int8(x, b, n, ORC_ROW, qx, sx);
  orc_quantize_int8(w, m, n, ORC_TENSOR, qw, &sw);
  orc_int8_gemm(qx, sx, 1, qw, &sw, 0, b, m, n, NULL, y);
  free(qx);
  free(qw);
  free(sx);
  return ORC_OK;
}

/* linear_backward {kSwitchBack, kInt8}, linear.cpp:199-248:
 * dX = int8_matmul_dequant(quantize_rowwise(G), quantize_tensorwise_transpose(W)) (:234-235)
 * dW = wgrad_full_precision(G, X) (:245). G b x m -> dX b x n, dW m x n. */
int orc_switchback_backward(const float* x, const float* w, const float* g, int64_t b, int64_t n,
                            int64_t m, float* dx, float* dw) {
  if (b == 0 || n == 0 || m == 0) return ORC_EMPTY;
  if (!all_finite(g, b * m)) return ORC_NONFINITE;
  int8_t* qg = (int8_t*)malloc((size_t)(b * m));
  int8_t* qwt = (int8_t*)malloc((size_t)(m * n));
  float* sg = (float*)malloc((size_t)b * sizeof(float));
  float sw;
  orc_quantize_int8(g, b, m, ORC_ROW, qg, sg);
  orc_quantize_tensorwise_transpose(w, m, n, qwt, &sw);
  orc_int8_gemm(qg, sg, 1, qwt, &sw, 0, b, n, m, NULL, dx);
  orc_wgrad_f32(g, x, b, m, n, dw);
  free(qg);
  free(qwt);
  free(sg);
  return ORC_OK;
}

/* ------------------------------------------------------- StableAdamW ----- */
/* debias, optimizer.cpp:63-68. */
double orc_debias(double beta, int64_t t) {
  if (beta == 0.0) return 0.0;
  double num = 1.0 - pow(beta, (double)(t - 1));
  double den = 1.0 - pow(beta, (double)t);
  return beta * num / den;
}

/* beta2_warmup, optimizer.cpp:44-49 (caller validates t >= 1, lambda > 0). */
double orc_beta2_warmup(int64_t t, double lambda) {
  double b = 1.0 - pow((double)t, -lambda);
  double cap = nextafter(1.0, 0.0);
  return b < cap ? b : cap;
}

/* compute_rms, optimizer.cpp:31-42. */
double orc_compute_rms(const float* g, const float* u, int64_t n, double eps) {
  double floor_ = eps * eps, acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double gi = (double)g[i];
    double ui = (double)u[i] > floor_ ? (double)u[i] : floor_;
    acc += gi * gi / ui;
  }
  return sqrt(acc / (double)n);
}

/* optimizer_step, optimizer.cpp:102-172. clipping: 0 none, 1 update_clip,
 * 2 grad_clip. alpha = lr_schedule(t) is passed in (the reference evaluates
 * its host std::function at :114). Tensors are processed in order; out_rms /
 * out_eta receive TensorStepInfo (optimizer.hpp:69-72). */
int orc_stableadamw_step(int ntensors, float** theta, const float** grad, float** v, float** u,
                         const int64_t* numel, double alpha, double beta1, double beta2,
                         double beta2_warmup_lambda, double eps, double weight_decay, int clipping,
                         double max_grad_norm, int64_t t, double* out_rms, double* out_eta) {
  if (t < 1) return ORC_BADARG;
  double b1 = orc_debias(beta1, t);
  double b2 = beta2_warmup_lambda > 0 ? orc_beta2_warmup(t, beta2_warmup_lambda) : orc_debias(beta2, t);
  double clip = 1.0;
  if (clipping == 2) { /* :121-131 */
    double ss = 0.0;
    for (int ti = 0; ti < ntensors; ++ti)
      for (int64_t i = 0; i < numel[ti]; ++i) ss += (double)grad[ti][i] * (double)grad[ti][i];
    double norm = sqrt(ss);
    if (norm > max_grad_norm) clip = max_grad_norm / norm;
  }
  for (int ti = 0; ti < ntensors; ++ti) {
    int64_t n = numel[ti];
    for (int64_t i = 0; i < n; ++i) { /* :142-146 */
      double g = (double)grad[ti][i] * clip;
      v[ti][i] = (float)(b1 * (double)v[ti][i] + (1.0 - b1) * g);
      u[ti][i] = (float)(b2 * (double)u[ti][i] + (1.0 - b2) * g * g);
    }
    double floor_ = eps * eps, acc = 0.0; /* :148-157 */
    for (int64_t i = 0; i < n; ++i) {
      double g = (double)grad[ti][i] * clip;
      double ui = (double)u[ti][i] > floor_ ? (double)u[ti][i] : floor_;
      acc += g * g / ui;
    }
    double rms = sqrt(acc / (double)n);
    double eta = clipping == 1 ? alpha / (rms > 1.0 ? rms : 1.0) : alpha; /* :159-160 */
    for (int64_t i = 0; i < n; ++i) { /* :162-167 */
      double th = (double)theta[ti][i];
      double upd = (double)v[ti][i] / (sqrt((double)u[ti][i]) + eps);
      theta[ti][i] = (float)(th - eta * weight_decay * th - eta * upd);
    }
    if (out_rms) out_rms[ti] = rms;
    if (out_eta) out_eta[ti] = eta;
  }
  return ORC_OK;
}

/* grad_clip_global_norm, optimizer.cpp:72-81 (standalone form, §8f "next"). */
int orc_grad_clip_global_norm(int ntensors, float** grads, const int64_t* numel, double max_norm) {
  if (max_norm <= 0) return ORC_BADARG;
  double ss = 0.0;
  for (int ti = 0; ti < ntensors; ++ti)
    for (int64_t i = 0; i < numel[ti]; ++i) ss += (double)grads[ti][i] * (double)grads[ti][i];
  double norm = sqrt(ss);
  if (!(norm > max_norm)) return ORC_OK;
  double c = max_norm / norm;
  for (int ti = 0; ti < ntensors; ++ti)
    for (int64_t i = 0; i < numel[ti]; ++i) grads[ti][i] = (float)((double)grads[ti][i] * c);
  return ORC_OK;
}
