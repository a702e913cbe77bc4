// capi.cu — the extern "C" boundary (include/switchback_b200.h).
//
// Argument checks reproduce the reference's std::invalid_argument conditions and
// messages ("<op>: <reason>", quantize.cpp:11-14, linear.cpp:55,73-74,80-81,87-93,
// 201-208, optimizer.cpp:104-112) as sb_status codes + sb_last_error() text.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sb_internal.h"

namespace sb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

sb_status fail(sb_status st, const char* op, const char* reason) {
  g_last_error = std::string(op) + ": " + reason;
  return st;
}

sb_status cuda_fail(const char* op, cudaError_t e) {
  g_last_error = std::string(op) + ": CUDA error: " + cudaGetErrorString(e);
  return SB_ERR_CUDA;
}

unsigned int* scratch(sb_handle h, size_t words) {
  const size_t bytes = words * sizeof(unsigned int);
  auto it = h->scratch.find(h->stream);
  if (it != h->scratch.end() && bytes <= it->second.second) return it->second.first;
  // a stream seen for the first time inside a graph capture cannot allocate (cudaMalloc /
  // cudaFree are illegal while capturing): it uses the buffer made at sb_create
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(h->stream, &cs);
  if (cs != cudaStreamCaptureStatusNone)
    return bytes <= h->capture_scratch_bytes ? h->capture_scratch : nullptr;
  auto& e = h->scratch[h->stream];
  if (e.first) {
    cudaStreamSynchronize(h->stream);
    cudaFree(e.first);
  }
  e = {nullptr, 0};
  const size_t want = std::max<size_t>(bytes, 65536);
  unsigned int* p = nullptr;
  if (cudaMalloc(&p, want) != cudaSuccess) return nullptr;
  e = {p, want};
  return p;
}

}  // namespace sb

namespace {

// Device constant 1.0f used as the "no scale" state of plain bf16 GEMMs.
__device__ float g_one = 1.0f;

struct Carve {
  uint8_t* base;
  size_t off = 0;
  template <typename T>
  T* take(size_t count) {
    off = (off + 255) & ~size_t(255);
    // a null base yields the offsets themselves (sb_linear_workspace_size / _layout)
    T* p = reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(base) + off);
    off += count * sizeof(T);
    return p;
  }
};

// Workspace carve-up shared by sb_linear_workspace_size / forward / backward.
struct LinearWs {
  int8_t* x_q;
  float* x_state;
  int8_t* w_q;
  int8_t* w_qt;
  float* w_state;  // 1 (tensor) or m (row-wise W, SwitchBackQ forward)
  float* wt_state; // n (column-wise W = rows of W^T, SwitchBackQ backward)
  unsigned int* words;  // absmax words: max(m, n, b) + 1
  int8_t* g_q;
  float* g_state;
  void* deq;       // SwitchBackM / fp8: dequantized operand buffer (b x n, dt)
  void* deq2;      // fp8 AllQuant / exact fp8: snapped G (b x m, dt)
  float* wdeq;     // exact fp8: snapped W (m x n, fp32)
  int8_t* gt_q;    // AllQuant int8: quantize_rowwise(G^T)  m x b
  float* gt_state;
  int8_t* xt_q;    // AllQuant int8: quantize_rowwise(X^T)  n x b
  float* xt_state;
  int64_t* raw64;  // AllQuant int8 under data parallelism: dW accumulators summed over ranks  m x n
  size_t total;
};

LinearWs carve(const sb_linear_mode& md, int64_t b, int64_t n, int64_t m, sb_dtype dt, void* base) {
  Carve c{static_cast<uint8_t*>(base)};
  LinearWs w{};
  const size_t es = dt == SB_BF16 ? 2 : 4;
  w.x_q = c.take<int8_t>(b * n);
  w.x_state = c.take<float>(b);
  w.w_q = c.take<int8_t>(m * n);
  w.w_qt = c.take<int8_t>(m * n);
  w.w_state = c.take<float>(std::max<int64_t>(m, 1));
  w.wt_state = c.take<float>(std::max<int64_t>(n, 1));
  w.words = c.take<unsigned int>(std::max(std::max(m, n), b) + 1);
  w.g_q = c.take<int8_t>(b * m);
  w.g_state = c.take<float>(b);
  const bool need_deq = md.variant == SB_SWITCHBACK_M || md.format == SB_FP8;
  w.deq = need_deq ? static_cast<void*>(c.take<uint8_t>(b * n * es)) : nullptr;
  w.deq2 = (md.format == SB_FP8 && (md.variant == SB_ALLQUANT || md.exact)) ? static_cast<void*>(c.take<uint8_t>(b * m * es))
                                                                           : nullptr;
  // exact fp8: the reference multiplies the dequantized (snapped) operands in fp32
  w.wdeq = (md.format == SB_FP8 && md.exact) ? c.take<float>(m * n) : nullptr;
  if (md.format == SB_INT8 && md.variant == SB_ALLQUANT) {
    w.gt_q = c.take<int8_t>(m * b);
    w.gt_state = c.take<float>(m);
    w.xt_q = c.take<int8_t>(n * b);
    w.xt_state = c.take<float>(n);
    w.raw64 = c.take<int64_t>(m * n);
  }
  w.total = c.off + 256;
  return w;
}

#define SB_TRY(expr)                       \
  do {                                     \
    sb_status _s = (expr);                 \
    if (_s != SB_OK) return _s;            \
  } while (0)
#define SB_TRYC(op, expr) SB_CUDA_CHECK(op, (expr))

__global__ void k_transpose_u8(const uint8_t* __restrict__ in, int64_t rows, int64_t cols, uint8_t* __restrict__ out) {
  __shared__ uint8_t t[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) t[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = t[threadIdx.x][i];
  }
}

sb_status transpose_u8(sb_handle h, const void* in, int64_t rows, int64_t cols, void* out) {
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  h->launches++;
  k_transpose_u8<<<grid, dim3(32, 8), 0, h->stream>>>(static_cast<const uint8_t*>(in), rows, cols,
                                                        static_cast<uint8_t*>(out));
  SB_LAUNCH_CHECK("transpose");
  return SB_OK;
}

bool float_dtype(sb_dtype dt) { return dt == SB_F32 || dt == SB_BF16; }

sb_status check_h(sb_handle h, const char* op) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null handle");
  cudaSetDevice(h->device);
  return SB_OK;
}

// ------------------------------------------------------------ quantize ops
// `word` must hold 4 device words.
sb_status q_tensorwise(sb_handle h, const void* x, sb_dtype dt, int64_t r, int64_t c, int64_t ldx, int8_t* q,
                       int64_t ldq, int8_t* qt, int64_t ldqt, float* state, unsigned int* word) {
  cudaError_t fe = cudaSuccess;
  static const bool fused = [] {  // SB_TW_FUSED=0: two launches (absmax, then quantize) -- A/B switch
    const char* e = std::getenv("SB_TW_FUSED");
    return !(e && e[0] == '0');
  }();
  if (fused && sb::launch_quantize_tensorwise_fused(h, x, dt, r, c, ldx, q, ldq, qt, ldqt, state, word, &fe)) {
    SB_TRYC("quantize_tensorwise", fe);
    return SB_OK;
  }
  SB_TRYC("quantize_tensorwise", sb::launch_absmax_tensor(h, x, dt, r, c, ldx, word));
  SB_TRYC("quantize_tensorwise", sb::launch_quantize_from_words(h, x, dt, r, c, ldx, word, 0, q, ldq, qt, ldqt, state));
  return SB_OK;
}

sb_status q_columnwise(sb_handle h, const void* x, sb_dtype dt, int64_t r, int64_t c, int64_t ldx, int8_t* q,
                       int64_t ldq, int8_t* qt, int64_t ldqt, float* state, unsigned int* words) {
  SB_TRYC("quantize_columnwise", sb::launch_absmax_columns(h, x, dt, r, c, ldx, words));
  SB_TRYC("quantize_columnwise", sb::launch_quantize_from_words(h, x, dt, r, c, ldx, words, 1, q, ldq, qt, ldqt, state));
  return SB_OK;
}

sb_status q_fp8(sb_handle h, const void* x, sb_dtype dt, int64_t r, int64_t c, int64_t ldx, int fmt, int axis,
                uint8_t* q, int64_t ldq, float* state, unsigned int* words) {
  const char* op = "quantize_fp8";
  cudaError_t fe = cudaSuccess;
  if (sb::launch_quantize_fp8_fast(h, x, dt, r, c, ldx, fmt, axis, words, q, ldq, state, true, &fe)) {
    SB_TRYC(op, fe);
    return SB_OK;
  }
  if (axis == SB_AXIS_ROW) {
    SB_TRYC(op, sb::launch_absmax_rows(h, x, dt, r, c, ldx, words));
  } else if (axis == SB_AXIS_COLUMN) {
    SB_TRYC(op, sb::launch_absmax_columns(h, x, dt, r, c, ldx, words));
  } else {
    SB_TRYC(op, sb::launch_absmax_tensor(h, x, dt, r, c, ldx, words));
  }
  if (sb::launch_quantize_fp8_fast(h, x, dt, r, c, ldx, fmt, axis, words, q, ldq, state, false, &fe)) {
    SB_TRYC(op, fe);
    return SB_OK;
  }
  SB_TRYC(op, sb::launch_quantize_fp8(h, x, dt, r, c, ldx, fmt, axis, words, q, ldq, state));
  return SB_OK;
}

// --------------------------------------------------------- plain bf16 GEMM
// (Standard-mode linear, fast path). a: [M x K] K-major or [K x M] MN-major, b likewise.
sb_status gemm_bf16(sb_handle h, const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K,
                    void* out, sb_dtype out_dt);

}  // namespace

// ======================================================================
extern "C" {

int sb_abi_version(void) { return SB_ABI_VERSION; }

sb_status sb_create(int device, sb_handle* out) {
  if (!out) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_create", "null out");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) return sb::fail(SB_ERR_CUDA, "sb_create", "no CUDA device");
  if (device < 0 || device >= count) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_create", "bad device");
  SB_CUDA_CHECK("sb_create", cudaSetDevice(device));
  cudaDeviceProp prop;
  SB_CUDA_CHECK("sb_create", cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return sb::fail(SB_ERR_UNSUPPORTED, "sb_create", "requires an sm_100 (B200) device");
  sb_handle h = new sb_handle_s();
  h->device = device;
  h->num_sms = prop.multiProcessorCount;
  if (cudaMalloc(&h->d_err, sizeof(uint32_t)) != cudaSuccess) {
    delete h;
    return sb::fail(SB_ERR_CUDA, "sb_create", "allocation failed");
  }
  cudaMemset(h->d_err, 0, sizeof(uint32_t));
  h->capture_scratch_bytes = 1 << 20;
  if (cudaMalloc(&h->capture_scratch, h->capture_scratch_bytes) != cudaSuccess) {
    cudaFree(h->d_err);
    delete h;
    return sb::fail(SB_ERR_CUDA, "sb_create", "allocation failed");
  }
  if (sb::build_gelu_lut(h) != cudaSuccess) {
    cudaFree(h->d_err);
    delete h;
    return sb::fail(SB_ERR_CUDA, "sb_create", "GELU table build failed");
  }
  cudaDeviceSynchronize();
  *out = h;
  return SB_OK;
}

sb_status sb_destroy(sb_handle h) {
  if (!h) return SB_OK;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  sb_dp_destroy(h);
  sb::dp_free_symmetric(h);
  if (h->d_err) cudaFree(h->d_err);
  if (h->gelu_lut) cudaFree(h->gelu_lut);
  for (auto& kv : h->scratch)
    if (kv.second.first) cudaFree(kv.second.first);
  if (h->capture_scratch) cudaFree(h->capture_scratch);
  for (int i = 0; i < 2; ++i) {
    if (h->dev_pool[i]) cudaFree(h->dev_pool[i]);
    if (h->pool_done[i]) cudaEventDestroy(h->pool_done[i]);
  }
  if (h->s_in) {
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_out);
    for (auto& row : h->hp_ev)
      for (auto& e : row) cudaEventDestroy(e);
    cudaEventDestroy(h->hp_start);
    cudaEventDestroy(h->hp_wready);
    cudaEventDestroy(h->hp_w1ready);
  }
  delete h;
  return SB_OK;
}

sb_status sb_set_stream(sb_handle h, void* s) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_set_stream", "null handle");
  h->stream = static_cast<cudaStream_t>(s);
  return SB_OK;
}

sb_status sb_set_gemm_path(sb_handle h, int path) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_set_gemm_path", "null handle");
  if (path < SB_GEMM_AUTO || path > SB_GEMM_2CTA_MC) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_set_gemm_path", "bad path");
  h->gemm_path = path;
  return SB_OK;
}

sb_status sb_synchronize(sb_handle h) {
  SB_TRY(check_h(h, "sb_synchronize"));
  SB_CUDA_CHECK("sb_synchronize", cudaStreamSynchronize(h->stream));
  uint32_t flags = 0;
  SB_CUDA_CHECK("sb_synchronize", cudaMemcpy(&flags, h->d_err, sizeof(flags), cudaMemcpyDeviceToHost));
  if (flags) {
    cudaMemset(h->d_err, 0, sizeof(uint32_t));
    return sb::fail(SB_ERR_NONFINITE, "switchback", "non-finite input");
  }
  return SB_OK;
}

uint32_t* sb_error_word(sb_handle h) { return h ? h->d_err : nullptr; }

const char* sb_last_error(void) { return sb::g_last_error.c_str(); }

uint64_t sb_launch_count(sb_handle h) { return h ? h->launches : 0; }

// ------------------------------------------------------------ quantize --
sb_status sb_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                              int8_t* q, int64_t ldq, float* state) {
  const char* op = "quantize_rowwise";
  SB_TRY(check_h(h, op));
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  if (!float_dtype(dt) || !x || !q || !state || ldx < cols || ldq < cols)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_TRYC(op, sb::launch_quantize_rowwise(h, x, dt, rows, cols, ldx, q, ldq, state));
  return SB_OK;
}

sb_status sb_quantize_columnwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state) {
  const char* op = "quantize_columnwise";
  SB_TRY(check_h(h, op));
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  if (!float_dtype(dt) || !x || (!q && !q_t) || !state || ldx < cols) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  unsigned int* words = sb::scratch(h, cols + 1);
  if (!words) return sb::fail(SB_ERR_CUDA, op, "scratch allocation failed (inside a graph capture: at most 256 K words)");
  return q_columnwise(h, x, dt, rows, cols, ldx, q, ldq, q_t, ldqt, state, words);
}

sb_status sb_quantize_tensorwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state) {
  const char* op = q ? "quantize_tensorwise" : "quantize_tensorwise_transpose";
  SB_TRY(check_h(h, op));
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  if (!float_dtype(dt) || !x || (!q && !q_t) || !state || ldx < cols) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  unsigned int* words = sb::scratch(h, 4);
  if (!words) return sb::fail(SB_ERR_CUDA, op, "scratch allocation failed (inside a graph capture: at most 256 K words)");
  return q_tensorwise(h, x, dt, rows, cols, ldx, q, ldq, q_t, ldqt, state, words);
}

sb_status sb_quantize_tensorwise_from_absmax(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                             int64_t ldx, const unsigned int* absmax_word, int8_t* q, int64_t ldq,
                                             int8_t* q_t, int64_t ldqt, float* state) {
  const char* op = "quantize_tensorwise";
  SB_TRY(check_h(h, op));
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  if (!float_dtype(dt) || !x || !absmax_word || (!q && !q_t) || !state || ldx < cols)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_TRYC(op, sb::launch_quantize_from_words(h, x, dt, rows, cols, ldx, absmax_word, 0, q, ldq, q_t, ldqt, state));
  return SB_OK;
}

sb_status sb_dequantize(sb_handle h, const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, const float* state,
                        sb_axis axis, void* y, sb_dtype ydt, int64_t ldy) {
  const char* op = "dequantize";
  SB_TRY(check_h(h, op));
  if (!q || !state || !y || !float_dtype(ydt) || axis < 0 || axis > 2)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "state length does not match axis");
  if (rows == 0 || cols == 0) return SB_OK;
  SB_TRYC(op, sb::launch_dequantize(h, q, rows, cols, ldq, state, axis, y, ydt, ldy));
  return SB_OK;
}

sb_status sb_quantize_fp8(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                          sb_fp8_format fmt, sb_axis axis, uint8_t* q, int64_t ldq, float* state) {
  const char* op = "quantize_fp8";
  SB_TRY(check_h(h, op));
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  if (!float_dtype(dt) || !x || !q || !state || (fmt != SB_E4M3 && fmt != SB_E5M2) || axis < 0 || axis > 2)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  unsigned int* words = sb::scratch(h, std::max(rows, cols) + 1);
  if (!words) return sb::fail(SB_ERR_CUDA, op, "scratch allocation failed (inside a graph capture: at most 256 K words)");
  return q_fp8(h, x, dt, rows, cols, ldx, fmt, axis, q, ldq, state, words);
}

sb_status sb_dequantize_fp8(sb_handle h, const uint8_t* q, int64_t rows, int64_t cols, int64_t ldq, sb_fp8_format fmt,
                            const float* state, sb_axis axis, void* y, sb_dtype ydt, int64_t ldy) {
  const char* op = "dequantize";
  SB_TRY(check_h(h, op));
  if (!q || !state || !y || !float_dtype(ydt)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (rows == 0 || cols == 0) return SB_OK;
  SB_TRYC(op, sb::launch_dequantize_fp8(h, q, rows, cols, ldq, fmt, state, axis, y, ydt, ldy));
  return SB_OK;
}

// ---------------------------------------------------------------- GEMM --
sb_status sb_gemm_i8(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sbp,
                     sb_scale_mode mode, int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt, int exact) {
  const char* op = mode == SB_SCALE_ROW_ROW ? "matmul_dequant_dual_rowwise" : "int8_matmul_dequant";
  SB_TRY(check_h(h, op));
  if (M < 0 || N < 0 || K < 0 || !qa || !qb || !out) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (mode != SB_SCALE_NONE && (!sa || !sbp)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "missing states");
  if (M == 0 || N == 0) return SB_OK;
  return sb::gemm_i8(h, qa, sa, qb, sbp, mode, M, N, K, out, out_dt, exact);
}

sb_status sb_gemm_i8_epilogue(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sbp,
                              sb_scale_mode mode, int64_t M, int64_t N, int64_t K, const float* bias,
                              const void* resid, int64_t ld_resid, void* out, sb_dtype out_dt, int exact) {
  const char* op = mode == SB_SCALE_ROW_ROW ? "matmul_dequant_dual_rowwise" : "int8_matmul_dequant";
  SB_TRY(check_h(h, op));
  if (M < 0 || N < 0 || K < 0 || !qa || !qb || !out || !sa || !sbp || mode == SB_SCALE_NONE ||
      (out_dt != SB_F32 && out_dt != SB_BF16) || (resid && ld_resid < N))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (M == 0 || N == 0) return SB_OK;
  return sb::gemm_i8(h, qa, sa, qb, sbp, mode, M, N, K, out, out_dt, exact, bias, resid, ld_resid);
}

sb_status sb_matmul_f32(sb_handle h, const float* a, const float* bt, int64_t r, int64_t c, int64_t k, float* y) {
  const char* op = "matmul";
  SB_TRY(check_h(h, op));
  if (!a || !bt || !y || r < 0 || c < 0 || k < 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "inner dimension mismatch");
  if (r == 0 || c == 0) return SB_OK;
  return sb::matmul_f32_seq(h, a, k, 1, bt, k, 1, r, c, k, y, 0);
}

sb_status sb_wgrad(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n, float* dw,
                   int exact, int accumulate) {
  const char* op = "linear_backward";
  SB_TRY(check_h(h, op));
  if (!g || !x || !dw || !float_dtype(dt) || b < 0 || m < 0 || n < 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (m == 0 || n == 0) return SB_OK;
  return sb::wgrad(h, g, x, dt, b, m, n, dw, exact, accumulate);
}

sb_status sb_wgrad_quantize_rowwise(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                    int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state) {
  const char* op = "linear_backward";
  SB_TRY(check_h(h, op));
  // an empty G is rejected as quantize_rowwise rejects it (require_quantizable, quantize.cpp:11-14)
  if (b <= 0 || m <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, "quantize_rowwise", "empty matrix");
  if (!float_dtype(dt) || n < 0 || ldq < m || !g || !g_q || !g_state || (n > 0 && (!x || !dw)))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  const sb::RowQuant rq{g_q, ldq, g_state};
  if (n == 0) {
    SB_TRYC(op, sb::launch_quantize_rowwise(h, g, dt, b, m, m, g_q, ldq, g_state));
    return SB_OK;
  }
  return sb::wgrad(h, g, x, dt, b, m, n, dw, 0, 0, &rq);
}

sb_status sb_gemm_fp8(sb_handle h, const uint8_t* qa, sb_fp8_format fa, const float* sa, sb_axis axa, const uint8_t* qb,
                      sb_fp8_format fb, const float* sbp, sb_axis axb, int64_t M, int64_t N, int64_t K, void* out,
                      sb_dtype out_dt) {
  const char* op = "fp8 matmul";
  SB_TRY(check_h(h, op));
  if (!qa || !qb || !sa || !sbp || !out) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (M == 0 || N == 0) return SB_OK;
  return sb::gemm_fp8(h, qa, fa, sa, axa, qb, fb, sbp, axb, M, N, K, out, out_dt);
}

// --------------------------------------------------------------- layer --
sb_status sb_linear_workspace_size(const sb_linear_mode* mode, int64_t b, int64_t n, int64_t m, size_t* bytes) {
  if (!mode || !bytes || b < 0 || n < 0 || m < 0)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "bad argument");
  *bytes = carve(*mode, b, n, m, SB_F32, nullptr).total;
  return SB_OK;
}

sb_status sb_linear_workspace_layout(const sb_linear_mode* mode, int64_t b, int64_t n, int64_t m,
                                     sb_linear_ws_layout* out) {
  if (!mode || !out || b < 0 || n < 0 || m < 0)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "bad argument");
  // the operand offsets do not depend on dt
  const LinearWs w = carve(*mode, b, n, m, SB_F32, nullptr);
  auto off = [](const void* p) { return static_cast<size_t>(reinterpret_cast<uintptr_t>(p)); };
  out->x_q = off(w.x_q);
  out->x_state = off(w.x_state);
  out->w_q = off(w.w_q);
  out->w_q_t = off(w.w_qt);
  out->w_state = off(w.w_state);
  out->g_q = off(w.g_q);
  out->g_state = off(w.g_state);
  out->total = w.total;
  return SB_OK;
}

static bool same_mode(const sb_linear_mode& a, const sb_linear_mode& b) {  // LinearMode ==, linear.cpp:27-32
  if (a.variant != b.variant || a.format != b.format || a.exact != b.exact) return false;
  if (a.format == SB_INT8) return true;
  return a.fp8_forward == b.fp8_forward && a.fp8_gradient == b.fp8_gradient;
}

}  // extern "C"

// linear_forward (+ optional fp32 column bias, fused into the int8 GEMM epilogue on the
// tensor-core path; added after the product on the others).
static sb_status linear_forward_impl(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                     const float* bias, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                                     sb_linear_ctx* ctx, void* workspace, size_t ws_bytes,
                                     const int8_t* xq_in = nullptr, const float* xs_in = nullptr,
                                     const void* resid = nullptr, const unsigned int* w_absmax = nullptr) {
  const char* op = "linear_forward";
  SB_TRY(check_h(h, op));
  if (!mode || !x || !w || !y || !float_dtype(dt)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (b <= 0 || n <= 0 || m <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty operand");  // linear.cpp:88
  const sb_linear_mode md = *mode;
  if (md.variant < SB_STANDARD || md.variant > SB_ALLQUANT || (md.format != SB_INT8 && md.format != SB_FP8))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "unknown mode");
  if (md.exact && dt != SB_F32) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "exact numerics need fp32 I/O");
  const LinearWs ws = carve(md, b, n, m, dt, workspace);
  if (md.variant != SB_STANDARD && (!workspace || ws_bytes < carve(md, b, n, m, dt, nullptr).total))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  if (ctx) {  // *ctx reset at entry, linear.cpp:116-119
    std::memset(ctx, 0, sizeof(*ctx));
    ctx->mode = md;
    ctx->b = b;
    ctx->n = n;
    ctx->m = m;
    ctx->dt = dt;
    ctx->x = x;
    ctx->w = w;
    ctx->workspace = workspace;
    ctx->workspace_bytes = ws_bytes;
  }
  const sb_dtype out_dt = dt;
  if (md.variant == SB_STANDARD) {  // linear.cpp:121-127
    if (md.exact || dt == SB_F32) {
      SB_TRY(sb::matmul_f32_seq(h, static_cast<const float*>(x), n, 1, static_cast<const float*>(w), n, 1, b, m, n,
                                static_cast<float*>(y), 0));
    } else {
      SB_TRY(gemm_bf16(h, x, false, w, false, b, m, n, y, out_dt));
    }
    if (bias) SB_TRYC(op, sb::launch_add_bias(h, y, out_dt, b, m, bias));
    if (resid) SB_TRYC(op, sb::launch_add_residual(h, y, out_dt, b, m, resid));
    if (ctx) ctx->valid = 1;
    return SB_OK;
  }
  if (md.format == SB_INT8) {
    // X quantized row-wise here, or already by its producer (fused activation + quantize)
    int8_t* xq = ws.x_q;
    float* xs = ws.x_state;
    if (xq_in) {
      xq = const_cast<int8_t*>(xq_in);
      xs = const_cast<float*>(xs_in);
    } else {
      SB_TRYC(op, sb::launch_quantize_rowwise(h, x, dt, b, n, n, xq, n, xs));
    }
    if (md.variant == SB_SWITCHBACK_Q) {
      // dual row-wise: Y = qrow(X) . qrow(W)^T (linear.cpp:131-132)
      SB_TRYC(op, sb::launch_quantize_rowwise(h, w, dt, m, n, n, ws.w_q, n, ws.w_state));
      SB_TRY(sb::gemm_i8(h, xq, xs, ws.w_q, ws.w_state, SB_SCALE_ROW_ROW, b, m, n, y, out_dt, md.exact, bias, resid, m));
    } else {
      // tensor-wise W, both layouts from one read; W^T payload cached for the backward. With
      // W's absmax already known (written by the optimizer step with the bf16 shadow), a single
      // quantize pass without the absmax pass.
      if (w_absmax)
        SB_TRYC(op, sb::launch_quantize_from_words(h, w, dt, m, n, n, w_absmax, 0, ws.w_q, n, ws.w_qt, m, ws.w_state));
      else
        SB_TRY(q_tensorwise(h, w, dt, m, n, n, ws.w_q, n, ws.w_qt, m, ws.w_state, ws.words));
      SB_TRY(sb::gemm_i8(h, xq, xs, ws.w_q, ws.w_state, SB_SCALE_ROW_TENSOR, b, m, n, y, out_dt, md.exact, bias, resid,
                         m));
    }
    if (ctx) {
      ctx->w_q_t = md.variant == SB_SWITCHBACK_Q ? nullptr : ws.w_qt;
      ctx->w_state = ws.w_state;
      if (md.variant == SB_SWITCHBACK_M) {  // linear.cpp:137-139: keep only the int8 tensors
        ctx->x_q = xq;
        ctx->x_state = xs;
        ctx->x = nullptr;
        ctx->w = nullptr;
      }
      ctx->valid = 1;
    }
    return SB_OK;
  }
  // fp8 (linear.cpp:148-163): snapped operands, tensor-core product
  const int ff = md.fp8_forward;
  const int ax = md.variant == SB_ALLQUANT ? SB_AXIS_TENSOR : SB_AXIS_ROW;   // fp8_activation_axis
  const int wx = md.variant == SB_SWITCHBACK_Q ? SB_AXIS_ROW : SB_AXIS_TENSOR;  // fp8_weight_axis
  uint8_t* xq = reinterpret_cast<uint8_t*>(ws.x_q);
  uint8_t* wq = reinterpret_cast<uint8_t*>(ws.w_q);
  SB_TRY(q_fp8(h, x, dt, b, n, n, ff, ax, xq, n, ws.x_state, ws.words));
  SB_TRY(q_fp8(h, w, dt, m, n, n, ff, wx, wq, n, ws.w_state, ws.words));
  if (md.exact) {  // matmul(dequantize(qx), dequantize(qw)), linear.cpp:151-153, sequential fp32
    SB_TRYC(op, sb::launch_dequantize_fp8(h, xq, b, n, n, ff, ws.x_state, ax, ws.deq, SB_F32, n));
    SB_TRYC(op, sb::launch_dequantize_fp8(h, wq, m, n, n, ff, ws.w_state, wx, ws.wdeq, SB_F32, n));
    SB_TRY(sb::matmul_f32_seq(h, static_cast<const float*>(ws.deq), n, 1, ws.wdeq, n, 1, b, m, n,
                              static_cast<float*>(y), 0));
  } else {
    SB_TRY(sb::gemm_fp8(h, xq, ff, ws.x_state, ax, wq, ff, ws.w_state, wx, b, m, n, y, out_dt));
  }
  if (bias) SB_TRYC(op, sb::launch_add_bias(h, y, out_dt, b, m, bias));
  if (resid) SB_TRYC(op, sb::launch_add_residual(h, y, out_dt, b, m, resid));
  if (ctx) {
    if (md.variant == SB_SWITCHBACK_M) {
      ctx->x_q = ws.x_q;
      ctx->x_state = ws.x_state;
      ctx->x = nullptr;
      ctx->w = nullptr;
    }
    ctx->w_state = ws.w_state;
    ctx->valid = 1;
  }
  return SB_OK;
}

extern "C" {

sb_status sb_linear_forward_ex(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                               const float* x_state, const void* w, const unsigned int* w_absmax, const float* bias,
                               const void* residual, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                               sb_linear_ctx* ctx, void* workspace, size_t ws_bytes) {
  if ((x_q == nullptr) != (x_state == nullptr))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "x_q and x_state go together");
  if ((x_q || w_absmax) && mode &&
      !(mode->format == SB_INT8 && (mode->variant == SB_SWITCHBACK || mode->variant == SB_SWITCHBACK_M ||
                                    (mode->variant == SB_SWITCHBACK_Q && !w_absmax))))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward",
                    "prequantized X needs a row-wise int8 variant; a W absmax needs tensor-wise W");
  return linear_forward_impl(h, mode, x, w, bias, dt, b, n, m, y, ctx, workspace, ws_bytes, x_q, x_state, residual,
                             w_absmax);
}

sb_status sb_linear_forward(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w, sb_dtype dt, int64_t b,
                            int64_t n, int64_t m, void* y, sb_linear_ctx* ctx, void* workspace, size_t ws_bytes) {
  return linear_forward_impl(h, mode, x, w, nullptr, dt, b, n, m, y, ctx, workspace, ws_bytes);
}

sb_status sb_linear_forward_bias(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                 const float* bias, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                                 sb_linear_ctx* ctx, void* workspace, size_t ws_bytes) {
  return linear_forward_impl(h, mode, x, w, bias, dt, b, n, m, y, ctx, workspace, ws_bytes);
}

sb_status sb_linear_forward_prequant(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                                     const float* x_state, const void* w, const float* bias, sb_dtype dt, int64_t b,
                                     int64_t n, int64_t m, void* y, sb_linear_ctx* ctx, void* workspace,
                                     size_t ws_bytes) {
  if (!mode || !x_q || !x_state || mode->format != SB_INT8 || mode->variant == SB_STANDARD ||
      mode->variant == SB_ALLQUANT || mode->exact)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "pre-quantized X needs an int8 row-wise variant");
  return linear_forward_impl(h, mode, x, w, bias, dt, b, n, m, y, ctx, workspace, ws_bytes, x_q, x_state);
}

sb_status sb_linear_forward_residual(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                                     const float* x_state, const void* w, const float* bias, const void* residual,
                                     sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y, sb_linear_ctx* ctx,
                                     void* workspace, size_t ws_bytes) {
  if (!residual) return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "null residual");
  if (x_q && (!x_state || !mode || mode->format != SB_INT8 || mode->variant == SB_STANDARD ||
              mode->variant == SB_ALLQUANT || mode->exact))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_forward", "pre-quantized X needs an int8 row-wise variant");
  return linear_forward_impl(h, mode, x, w, bias, dt, b, n, m, y, ctx, workspace, ws_bytes, x_q, x_state, residual);
}

}  // extern "C"

static sb_status linear_backward_impl(sb_handle h, const sb_linear_mode* mode, const sb_linear_ctx* ctx, const void* g,
                                      void* dx, float* dw, int dw_accumulate, const int8_t* gq_in = nullptr,
                                      const float* gs_in = nullptr) {
  const char* op = "linear_backward";
  SB_TRY(check_h(h, op));
  if (!mode || !ctx || !ctx->valid || !g || !dx || !dw) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (!same_mode(*mode, ctx->mode))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "context was produced by a different mode");  // linear.cpp:201-202
  const sb_linear_mode md = ctx->mode;
  const int64_t b = ctx->b, n = ctx->n, m = ctx->m;
  const sb_dtype dt = ctx->dt;
  const LinearWs ws = carve(md, b, n, m, dt, ctx->workspace);
  const int exact = md.exact;

  if (md.variant == SB_STANDARD) {  // linear.cpp:210-214
    if (exact || dt == SB_F32) {
      // x_grad = matmul(G, W^T^T) : dx[i][j] = sum_p g[i][p] * w[p][j]
      SB_TRY(sb::matmul_f32_seq(h, static_cast<const float*>(g), m, 1, static_cast<const float*>(ctx->w), 1, n, b, n, m,
                                static_cast<float*>(dx), 0));
    } else {
      SB_TRY(gemm_bf16(h, g, false, ctx->w, true, b, n, m, dx, dt));
    }
    return sb::wgrad(h, g, ctx->x, dt, b, m, n, dw, exact, dw_accumulate);
  }

  if (md.format == SB_INT8) {
    // G quantized row-wise here, or already by its producer (fused GELU backward + quantize)
    int8_t* gq = ws.g_q;
    float* gs = ws.g_state;
    bool dw_done = false;
    if (gq_in) {
      gq = const_cast<int8_t*>(gq_in);
      gs = const_cast<float*>(gs_in);
    } else if (md.variant == SB_SWITCHBACK) {
      // dW = G^T X first, with the row-wise quantize of G riding in the same launch (the dW
      // kernel's idle warps, tc_dw_wide.cuh); dX below consumes G_q. Both only read G
      // (linear.cpp:232-245), so the order does not change any result.
      const sb::RowQuant rq{gq, m, gs};
      SB_TRY(sb::wgrad(h, g, ctx->x, dt, b, m, n, dw, exact, dw_accumulate, &rq));
      dw_done = true;
    } else {
      SB_TRYC(op, sb::launch_quantize_rowwise(h, g, dt, b, m, m, gq, m, gs));
    }
    if (md.variant == SB_SWITCHBACK_Q) {
      // column-wise quantize-transpose of W: per-row states of W^T (linear.cpp:226-229)
      SB_TRY(q_columnwise(h, ctx->w, dt, m, n, n, nullptr, 0, ws.w_qt, m, ws.wt_state, ws.words));
      SB_TRY(sb::gemm_i8(h, gq, gs, ws.w_qt, ws.wt_state, SB_SCALE_ROW_ROW, b, n, m, dx, dt, exact));
    } else {
      // W^T payload from the forward (== quantize_tensorwise_transpose(W), linear_test.cpp:252-264)
      SB_TRY(sb::gemm_i8(h, gq, gs, ctx->w_q_t, ctx->w_state, SB_SCALE_ROW_TENSOR, b, n, m, dx, dt, exact));
    }
    if (md.variant == SB_ALLQUANT) {
      // dW = dual_rowwise(qrow(G^T), qrow(X^T)) with K = b (linear.cpp:239-241)
      if (dw_accumulate) return sb::fail(SB_ERR_UNSUPPORTED, op, "AllQuant dW does not accumulate");
      if (sb::dp_active(h)) {
        // token-sharded: the rows of G^T / X^T span every rank's tokens, so the per-feature
        // absmax is a max over ranks, and dW's integer accumulators are summed over ranks
        // before the one dequantization (bit-identical to the single-GPU product)
        return sb::dp_allquant_dw(h, g, ctx->x, dt, b, n, m, ws.gt_q, ws.gt_state, ws.xt_q, ws.xt_state, ws.words,
                                  ws.raw64, dw);
      }
      SB_TRY(q_columnwise(h, g, dt, b, m, m, nullptr, 0, ws.gt_q, b, ws.gt_state, ws.words));
      SB_TRY(q_columnwise(h, ctx->x, dt, b, n, n, nullptr, 0, ws.xt_q, b, ws.xt_state, ws.words));
      return sb::gemm_i8(h, ws.gt_q, ws.gt_state, ws.xt_q, ws.xt_state, SB_SCALE_ROW_ROW, m, n, b, dw, SB_F32, exact);
    }
    if (md.variant == SB_SWITCHBACK_M) {
      // dW on the dequantized saved activations (linear.cpp:243)
      SB_TRYC(op, sb::launch_dequantize(h, ctx->x_q, b, n, n, ctx->x_state, SB_AXIS_ROW, ws.deq, dt, n));
      return sb::wgrad(h, g, ws.deq, dt, b, m, n, dw, exact, dw_accumulate);
    }
    if (dw_done) return SB_OK;
    return sb::wgrad(h, g, ctx->x, dt, b, m, n, dw, exact, dw_accumulate);  // linear.cpp:245
  }

  // fp8 backward (linear.cpp:250-277)
  const int ff = md.fp8_forward, fg = md.fp8_gradient;
  uint8_t* wqt = reinterpret_cast<uint8_t*>(ws.w_qt);
  uint8_t* wq = reinterpret_cast<uint8_t*>(ws.w_q);
  const float* wt_state;
  int wt_axis;
  if (md.variant == SB_SWITCHBACK_M) {  // transpose of the saved tensor-wise payload
    SB_TRY(transpose_u8(h, wq, m, n, wqt));
    wt_state = ctx->w_state;
    wt_axis = SB_AXIS_TENSOR;
  } else if (md.variant == SB_SWITCHBACK_Q) {  // per-column states of W
    SB_TRY(q_fp8(h, ctx->w, dt, m, n, n, ff, SB_AXIS_COLUMN, wq, n, ws.wt_state, ws.words));
    SB_TRY(transpose_u8(h, wq, m, n, wqt));
    wt_state = ws.wt_state;
    wt_axis = SB_AXIS_ROW;
  } else {
    // the forward's tensor-wise payload of W (ws.w_q, state ws.w_state) is still in the
    // workspace and W is unmodified (ctx contract), so re-quantizing it (linear.cpp:259-261)
    // would reproduce it bit for bit: transpose it instead
    SB_TRY(transpose_u8(h, wq, m, n, wqt));
    wt_state = ws.w_state;
    wt_axis = SB_AXIS_TENSOR;
  }
  const int gx = md.variant == SB_ALLQUANT ? SB_AXIS_TENSOR : SB_AXIS_ROW;
  uint8_t* gq = reinterpret_cast<uint8_t*>(ws.g_q);
  SB_TRY(q_fp8(h, g, dt, b, m, m, fg, gx, gq, m, ws.g_state, ws.words));
  if (exact) {  // x_grad = matmul(g_snap, w_snap_t), linear.cpp:266, sequential fp32
    SB_TRYC(op, sb::launch_dequantize_fp8(h, gq, b, m, m, fg, ws.g_state, gx, ws.deq2, SB_F32, m));
    SB_TRYC(op, sb::launch_dequantize_fp8(h, reinterpret_cast<const uint8_t*>(wqt), n, m, m, ff, wt_state, wt_axis,
                                          ws.wdeq, SB_F32, m));
    SB_TRY(sb::matmul_f32_seq(h, static_cast<const float*>(ws.deq2), m, 1, ws.wdeq, m, 1, b, n, m,
                              static_cast<float*>(dx), 0));
  } else {
    SB_TRY(sb::gemm_fp8(h, gq, fg, ws.g_state, gx, wqt, ff, wt_state, wt_axis, b, n, m, dx, dt));
  }
  if (md.variant == SB_ALLQUANT) {
    // wgrad over snapped G and snapped (tensor-wise) X
    SB_TRYC(op, sb::launch_dequantize_fp8(h, gq, b, m, m, fg, ws.g_state, gx, ws.deq2, dt, m));
    uint8_t* xq = reinterpret_cast<uint8_t*>(ws.x_q);
    SB_TRY(q_fp8(h, ctx->x, dt, b, n, n, ff, SB_AXIS_TENSOR, xq, n, ws.x_state, ws.words));
    SB_TRYC(op, sb::launch_dequantize_fp8(h, xq, b, n, n, ff, ws.x_state, SB_AXIS_TENSOR, ws.deq, dt, n));
    return sb::wgrad(h, ws.deq2, ws.deq, dt, b, m, n, dw, exact, dw_accumulate);
  }
  if (md.variant == SB_SWITCHBACK_M) {
    SB_TRYC(op, sb::launch_dequantize_fp8(h, reinterpret_cast<const uint8_t*>(ctx->x_q), b, n, n, ff, ctx->x_state,
                                          SB_AXIS_ROW, ws.deq, dt, n));
    return sb::wgrad(h, g, ws.deq, dt, b, m, n, dw, exact, dw_accumulate);
  }
  return sb::wgrad(h, g, ctx->x, dt, b, m, n, dw, exact, dw_accumulate);
}

extern "C" {

sb_status sb_linear_backward(sb_handle h, const sb_linear_mode* mode, const sb_linear_ctx* ctx, const void* g, void* dx,
                             float* dw, int dw_accumulate) {
  return linear_backward_impl(h, mode, ctx, g, dx, dw, dw_accumulate);
}

sb_status sb_linear_backward_prequant(sb_handle h, const sb_linear_mode* mode, const sb_linear_ctx* ctx, const void* g,
                                      const int8_t* g_q, const float* g_state, void* dx, float* dw, int dw_accumulate) {
  if (!mode || !g_q || !g_state || mode->format != SB_INT8 || mode->variant == SB_STANDARD ||
      mode->variant == SB_ALLQUANT || mode->exact)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "linear_backward", "pre-quantized G needs an int8 row-wise variant");
  return linear_backward_impl(h, mode, ctx, g, dx, dw, dw_accumulate, g_q, g_state);
}

sb_status sb_gelu_quantize_rowwise(sb_handle h, const void* pre, sb_dtype dt, int64_t rows, int64_t cols, void* act,
                                   int8_t* q, float* state) {
  const char* op = "gelu_quantize_rowwise";
  SB_TRY(check_h(h, op));
  if (!pre || !act || !q || !state || dt != SB_BF16) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (bf16 only)");
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  SB_TRYC(op, sb::launch_act_quantize_rowwise(h, 0, pre, nullptr, rows, cols, act, q, state));
  return SB_OK;
}

sb_status sb_gelu_backward_quantize_rowwise(sb_handle h, const void* dact, const void* pre, sb_dtype dt, int64_t rows,
                                            int64_t cols, void* g, int8_t* q, float* state) {
  const char* op = "gelu_backward_quantize_rowwise";
  SB_TRY(check_h(h, op));
  if (!dact || !pre || !g || !q || !state || dt != SB_BF16)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (bf16 only)");
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  SB_TRYC(op, sb::launch_act_quantize_rowwise(h, 1, dact, pre, rows, cols, g, q, state));
  return SB_OK;
}

sb_status sb_heads_pack_quantize(sb_handle h, const void* const* dqkv, const int64_t* strides, int64_t B, int64_t S,
                                 int H, int Dh, void* g, int8_t* const* q, float* const* state) {
  const char* op = "heads_pack_quantize";
  SB_TRY(check_h(h, op));
  if (!dqkv || !strides || !g || !q || !state || B <= 0 || S <= 0 || H <= 0 || Dh <= 0)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  for (int i = 0; i < 3; ++i)
    if (!dqkv[i] || !q[i] || !state[i]) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  const cudaError_t e = sb::launch_heads_pack_quantize(h, dqkv, strides, B, S, H, Dh, g, q, state);
  if (e == cudaErrorNotSupported)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "bf16, H * Dh <= 2048, Dh % 8 == 0, 16-byte aligned heads");
  SB_TRYC(op, e);
  return SB_OK;
}

sb_status sb_layernorm_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                        const float* gamma, const float* beta, float eps, void* out, int8_t* q,
                                        float* state, float* mean, float* rstd) {
  const char* op = "layernorm_quantize_rowwise";
  SB_TRY(check_h(h, op));
  if (!x || !gamma || !beta || !out || !q || !state || !mean || !rstd || dt != SB_BF16)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (bf16 only)");
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  const cudaError_t e = sb::launch_ln_quantize_rowwise(h, x, rows, cols, gamma, beta, eps, out, q, state, mean, rstd);
  if (e == cudaErrorNotSupported)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "rows of <= 2048 columns, multiple of 8, 16-byte aligned");
  SB_TRYC(op, e);
  return SB_OK;
}

sb_status sb_layernorm_backward_workspace_size(sb_handle h, int64_t cols, size_t* bytes) {
  SB_TRY(check_h(h, "layernorm_backward"));
  if (!bytes || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, "layernorm_backward", "bad argument");
  *bytes = static_cast<size_t>(sb::ln_backward_blocks(h)) * 2 * static_cast<size_t>(cols) * sizeof(float);
  return SB_OK;
}

sb_status sb_layernorm_backward(sb_handle h, const void* dh, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                const float* mean, const float* rstd, const float* gamma, void* dx, float* dgamma,
                                float* dbeta, void* workspace, size_t workspace_bytes) {
  const char* op = "layernorm_backward";
  SB_TRY(check_h(h, op));
  if (!dh || !x || !mean || !rstd || !gamma || !dx || !workspace || dt != SB_BF16)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (bf16 only)");
  if (rows <= 0 || cols <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty matrix");
  size_t need = 0;
  SB_TRY(sb_layernorm_backward_workspace_size(h, cols, &need));
  if (workspace_bytes < need) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  const cudaError_t e = sb::launch_ln_backward(h, dh, x, rows, cols, mean, rstd, gamma, dx, dgamma, dbeta,
                                               static_cast<float*>(workspace));
  if (e == cudaErrorNotSupported)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "rows of <= 1280 columns, multiple of 8, 16-byte aligned");
  SB_TRYC(op, e);
  return SB_OK;
}

// ------------------------------------------------- host-buffer pipeline --
// Copy streams, per-slot events and the two alternating device pools of the host-buffer
// entries; created on first use. *pi = the pool this call owns (big enough for `need`).
static sb_status host_pool_acquire(sb_handle h, const char* op, size_t need, int* pi_out) {
  if (!h->s_in) {
    SB_CUDA_CHECK(op, cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
    SB_CUDA_CHECK(op, cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    for (auto& row : h->hp_ev)
      for (auto& e : row) SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&h->hp_start, cudaEventDisableTiming));
    SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&h->hp_wready, cudaEventDisableTiming));
    SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&h->hp_w1ready, cudaEventDisableTiming));
    for (auto& e : h->pool_done) SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int pi = h->pool_next;
  h->pool_next ^= 1;
  if (need > h->dev_pool_bytes[pi]) {
    if (h->dev_pool[pi]) {
      cudaDeviceSynchronize();  // the pool's previous call may still be in flight
      cudaFree(h->dev_pool[pi]);
    }
    h->dev_pool[pi] = nullptr;
    h->dev_pool_bytes[pi] = 0;
    h->pool_used[pi] = false;
    SB_CUDA_CHECK(op, cudaMalloc(&h->dev_pool[pi], need));
    h->dev_pool_bytes[pi] = need;
  }
  *pi_out = pi;
  return SB_OK;
}

// Stream order at the start of a host-pipeline call. s_in only writes this call's private
// pool: it does not wait for earlier compute, so an async call's first chunks stream in while
// the previous call drains.
static void host_pool_begin(sb_handle h, int pi) {
  cudaEventRecord(h->hp_start, h->stream);
  cudaStreamWaitEvent(h->s_out, h->hp_start, 0);
  if (h->pool_used[pi]) {  // this pool's previous call (two calls ago) has fully drained
    cudaStreamWaitEvent(h->s_in, h->pool_done[pi], 0);
    cudaStreamWaitEvent(h->stream, h->pool_done[pi], 0);
  }
}

// Slot count / chunk rows of the host pipelines (SB_HOST_SLOTS / SB_HOST_CHUNK override).
static void host_chunking(int64_t b, int64_t def_chunk, int* ns, int64_t* chunk) {
  const char* ce = std::getenv("SB_HOST_CHUNK");
  const char* se = std::getenv("SB_HOST_SLOTS");
  *ns = se ? std::max(2, std::min(8, std::atoi(se))) : 4;
  *chunk = std::min<int64_t>(b, ce ? std::max<int64_t>(128, std::atoll(ce)) : def_chunk);
}

// switchback_fwd_bwd over host memory: W is quantized once; token rows stream through in
// chunks. Three streams: h2d copies, compute (the handle stream), d2h copies, so PCIe
// transfers of chunk i+1 / i-1 overlap the kernels of chunk i. dW accumulates on the single
// compute stream in chunk order (deterministic).
static sb_status fwd_bwd_host_enqueue(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                      const void* g, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y, void* dx,
                                      float* dw) {
  const char* op = "switchback_fwd_bwd";
  SB_TRY(check_h(h, op));
  if (!mode || !x || !w || !g || !y || !dx || !dw || !float_dtype(dt)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (b <= 0 || n <= 0 || m <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty operand");
  if (mode->variant != SB_SWITCHBACK || mode->format != SB_INT8)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "host pipeline implements SwitchBack int8");
  const size_t es = sb::dt_size(dt);
  // Token rows stream through NS slots of `chunk` rows: H2D of chunk i+2 | kernels of chunk i |
  // D2H of chunk i-1 run concurrently; Y of a chunk is copied out as soon as its forward GEMM
  // is done, dX after the backward. Small chunks keep the un-overlapped pipeline fill (first
  // H2D) and drain (last D2H, the dW copy) short; 2048-row chunks x 4 slots measured best
  // (tools/e2e_sweep.py: 39.7 ms per C2 step async, against 40.4 ms at 4096 x 3).
  // SB_HOST_CHUNK / SB_HOST_SLOTS override the defaults (measurement knobs).
  int NS = 4;
  int64_t chunk = 2048;
  host_chunking(b, 2048, &NS, &chunk);
  // device layout: W, W_q, W_qT, dW, states/words, NS x {x, g, y, dx, x_q, g_q, x states, g states}
  Carve c{nullptr};
  auto layout = [&](Carve& cv, void** P) {
    P[0] = cv.take<uint8_t>(m * n * es);
    P[1] = cv.take<int8_t>(m * n);
    P[2] = cv.take<int8_t>(m * n);
    P[3] = cv.take<float>(m * n);
    P[4] = cv.take<float>(8);
    P[5] = cv.take<unsigned int>(8);
    for (int s = 0; s < NS; ++s) {
      P[6 + 8 * s + 0] = cv.take<uint8_t>(chunk * n * es);
      P[6 + 8 * s + 1] = cv.take<uint8_t>(chunk * m * es);
      P[6 + 8 * s + 2] = cv.take<uint8_t>(chunk * m * es);
      P[6 + 8 * s + 3] = cv.take<uint8_t>(chunk * n * es);
      P[6 + 8 * s + 4] = cv.take<int8_t>(chunk * n);
      P[6 + 8 * s + 5] = cv.take<int8_t>(chunk * m);
      P[6 + 8 * s + 6] = cv.take<float>(chunk);
      P[6 + 8 * s + 7] = cv.take<float>(chunk);
    }
  };
  void* P[6 + 8 * 8];
  layout(c, P);
  const size_t need = c.off + 256;
  int pi = 0;
  SB_TRY(host_pool_acquire(h, op, need, &pi));
  Carve c2{static_cast<uint8_t*>(h->dev_pool[pi])};
  layout(c2, P);
  void* dW_ = P[0];
  int8_t* wq = static_cast<int8_t*>(P[1]);
  int8_t* wqt = static_cast<int8_t*>(P[2]);
  float* dwd = static_cast<float*>(P[3]);
  float* wstate = static_cast<float*>(P[4]);
  unsigned int* words = static_cast<unsigned int*>(P[5]);
  cudaEvent_t* ev_in = h->hp_ev[0];
  cudaEvent_t* ev_y = h->hp_ev[1];
  cudaEvent_t* ev_comp = h->hp_ev[2];
  cudaEvent_t* ev_out = h->hp_ev[3];
  cudaEvent_t* ev_x = h->hp_ev[4];

  cudaStream_t comp = h->stream, s_in = h->s_in, s_out = h->s_out;
  host_pool_begin(h, pi);
  sb_status st = SB_OK;
  const int64_t nchunks = (b + chunk - 1) / chunk;
  // a chunk's x (ev_x: its forward may start), then its g (ev_in: its backward may start)
  auto h2d = [&](int64_t i) {
    const int s = static_cast<int>(i % NS);
    const int64_t r0 = i * chunk, rows = std::min(chunk, b - r0);
    if (i >= NS) cudaStreamWaitEvent(s_in, ev_comp[s], 0);  // slot's x, g consumed by chunk i-NS
    cudaMemcpyAsync(P[6 + 8 * s + 0], static_cast<const uint8_t*>(x) + r0 * n * es, rows * n * es, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev_x[s], s_in);
    cudaMemcpyAsync(P[6 + 8 * s + 1], static_cast<const uint8_t*>(g) + r0 * m * es, rows * m * es, cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev_in[s], s_in);
  };
  // W in, quantized once (both layouts), while the first chunks stream in
  h2d(0);
  cudaMemcpyAsync(dW_, w, m * n * es, cudaMemcpyHostToDevice, comp);
  st = q_tensorwise(h, dW_, dt, m, n, n, wq, n, wqt, m, wstate, words);
  for (int64_t i = 1; i < std::min<int64_t>(NS - 1, nchunks); ++i) h2d(i);
  for (int64_t i = 0; i < nchunks && st == SB_OK; ++i) {
    const int s = static_cast<int>(i % NS);
    const int64_t r0 = i * chunk, rows = std::min(chunk, b - r0);
    if (i + NS - 1 < nchunks) h2d(i + NS - 1);
    cudaStreamWaitEvent(comp, ev_x[s], 0);
    if (i >= NS) cudaStreamWaitEvent(comp, ev_out[s], 0);  // slot's y, dx copied out
    void* xd = P[6 + 8 * s + 0];
    void* gd = P[6 + 8 * s + 1];
    void* yd = P[6 + 8 * s + 2];
    void* dxd = P[6 + 8 * s + 3];
    int8_t* xq = static_cast<int8_t*>(P[6 + 8 * s + 4]);
    int8_t* gq = static_cast<int8_t*>(P[6 + 8 * s + 5]);
    float* xs = static_cast<float*>(P[6 + 8 * s + 6]);
    float* gs = static_cast<float*>(P[6 + 8 * s + 7]);
    if (sb::launch_quantize_rowwise(h, xd, dt, rows, n, n, xq, n, xs) != cudaSuccess) st = sb::cuda_fail(op, cudaGetLastError());
    if (st == SB_OK) st = sb::gemm_i8(h, xq, xs, wq, wstate, SB_SCALE_ROW_TENSOR, rows, m, n, yd, dt, mode->exact);
    cudaEventRecord(ev_y[s], comp);
    // backward: dW += G^T X with G's row-wise quantize in the same launch, then the dX GEMM
    cudaStreamWaitEvent(comp, ev_in[s], 0);
    const sb::RowQuant rq{gq, m, gs};
    if (st == SB_OK) st = sb::wgrad(h, gd, xd, dt, rows, m, n, dwd, mode->exact, i > 0, &rq);
    if (st == SB_OK) st = sb::gemm_i8(h, gq, gs, wqt, wstate, SB_SCALE_ROW_TENSOR, rows, n, m, dxd, dt, mode->exact);
    cudaEventRecord(ev_comp[s], comp);
    cudaStreamWaitEvent(s_out, ev_y[s], 0);
    cudaMemcpyAsync(static_cast<uint8_t*>(y) + r0 * m * es, yd, rows * m * es, cudaMemcpyDeviceToHost, s_out);
    cudaStreamWaitEvent(s_out, ev_comp[s], 0);
    cudaMemcpyAsync(static_cast<uint8_t*>(dx) + r0 * n * es, dxd, rows * n * es, cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(ev_out[s], s_out);
  }
  // dW leaves on the D2H stream after the last chunk's compute; the event marks the pool free.
  // The per-slot events are reused by the next call, so later calls must not wait on this
  // call's recordings: every stream of the next call first waits on hp_start (recorded on
  // comp) and comp waits here for this call's D2H before anything else is enqueued on it.
  cudaEventRecord(ev_comp[0], comp);
  cudaStreamWaitEvent(s_out, ev_comp[0], 0);
  cudaMemcpyAsync(dw, dwd, m * n * sizeof(float), cudaMemcpyDeviceToHost, s_out);
  cudaEventRecord(h->pool_done[pi], s_out);
  h->pool_used[pi] = true;
  return st;
}


// Two chained SwitchBack int8 linears over host memory — the MLP block of model.cpp:324-329
// (fc1: n -> hd, optional GELU, fc2: hd -> m) and its backward (model.cpp:351-360) — with the
// hidden activation and its gradient kept on the device. Per token chunk (rows are
// independent in every op but the W quantize and the dW sums):
//   X_c -> q -> fc1 GEMM -> P_c [-> GELU] = A_c -> q -> fc2 GEMM -> Y_c            (Y_c out)
//   G_c -> dW2 += G_c^T A_c (G_c's quantize in the same launch) -> dX2 GEMM -> dA_c
//   [dA_c * GELU'(P_c)] = G1_c -> dW1 += G1_c^T X_c (+ quantize G1_c) -> dX GEMM -> dX_c (out)
// dW1 / dW2 accumulate in chunk order on the compute stream (deterministic) and leave last.
static sb_status mlp_host_enqueue(sb_handle h, const sb_linear_mode* mode, int activation, const void* x,
                                  const void* w1, const void* w2, const void* g, sb_dtype dt, int64_t b, int64_t n,
                                  int64_t hd, int64_t m, void* y, void* dx, float* dw1, float* dw2) {
  const char* op = "switchback_mlp_fwd_bwd";
  SB_TRY(check_h(h, op));
  if (!mode || !x || !w1 || !w2 || !g || !y || !dx || !dw1 || !dw2 || !float_dtype(dt))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (b <= 0 || n <= 0 || hd <= 0 || m <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty operand");
  if (mode->variant != SB_SWITCHBACK || mode->format != SB_INT8)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "host pipeline implements SwitchBack int8");
  if (activation != SB_ACT_NONE && activation != SB_ACT_GELU)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "unknown activation");
  if (activation == SB_ACT_GELU && (dt != SB_BF16 || mode->exact))
    return sb::fail(SB_ERR_UNSUPPORTED, op, "GELU runs on the bf16 performance path");
  const size_t es = sb::dt_size(dt);
  const bool gelu = activation == SB_ACT_GELU;
  // 4096-row chunks (1024-row first chunk, halving end taper) measured best at the C2 shape once
  // a chunk's forward waits only for its x (tools/mlp_e2e_sweep.py, one box, alternating runs):
  // 8.87 ms per call against 9.03 / 9.27 / 9.39 / 9.45 ms at 3584 / 4608 / 5120 / 8192 rows and
  // 9.82 ms at 2048 (with both x and g awaited, 8192 had been best)
  int NS = 4;
  int64_t chunk = 4096;
  host_chunking(b, 4096, &NS, &chunk);
  // pool layout: weights {W1, W2, payloads (both layouts), states, words}, dW1, dW2; the
  // compute-only chunk buffers once (one compute stream); NS copy slots {x, g, y, dx}
  enum { W1, W2, W1Q, W1QT, W2Q, W2QT, WST1, WST2, WRD1, WRD2, DW1, DW2, XQ, XS, PRE, ACT, HQ, HS, GQ, GS, DA,
         G1, G1Q, G1S, NFIX };
  Carve c{nullptr};
  auto layout = [&](Carve& cv, void** P) {
    P[W1] = cv.take<uint8_t>(hd * n * es);
    P[W2] = cv.take<uint8_t>(m * hd * es);
    P[W1Q] = cv.take<int8_t>(hd * n);
    P[W1QT] = cv.take<int8_t>(hd * n);
    P[W2Q] = cv.take<int8_t>(m * hd);
    P[W2QT] = cv.take<int8_t>(m * hd);
    P[WST1] = cv.take<float>(8);
    P[WST2] = cv.take<float>(8);
    P[WRD1] = cv.take<unsigned int>(8);
    P[WRD2] = cv.take<unsigned int>(8);
    P[DW1] = cv.take<float>(hd * n);
    P[DW2] = cv.take<float>(m * hd);
    P[XQ] = cv.take<int8_t>(chunk * n);
    P[XS] = cv.take<float>(chunk);
    P[PRE] = cv.take<uint8_t>(chunk * hd * es);
    P[ACT] = gelu ? cv.take<uint8_t>(chunk * hd * es) : P[PRE];
    P[HQ] = cv.take<int8_t>(chunk * hd);
    P[HS] = cv.take<float>(chunk);
    P[GQ] = cv.take<int8_t>(chunk * m);
    P[GS] = cv.take<float>(chunk);
    P[DA] = cv.take<uint8_t>(chunk * hd * es);
    P[G1] = gelu ? cv.take<uint8_t>(chunk * hd * es) : P[DA];
    P[G1Q] = cv.take<int8_t>(chunk * hd);
    P[G1S] = cv.take<float>(chunk);
    for (int s = 0; s < NS; ++s) {
      P[NFIX + 4 * s + 0] = cv.take<uint8_t>(chunk * n * es);
      P[NFIX + 4 * s + 1] = cv.take<uint8_t>(chunk * m * es);
      P[NFIX + 4 * s + 2] = cv.take<uint8_t>(chunk * m * es);
      P[NFIX + 4 * s + 3] = cv.take<uint8_t>(chunk * n * es);
    }
  };
  void* P[NFIX + 4 * 8];
  layout(c, P);
  int pi = 0;
  SB_TRY(host_pool_acquire(h, op, c.off + 256, &pi));
  Carve c2{static_cast<uint8_t*>(h->dev_pool[pi])};
  layout(c2, P);
  auto I8 = [&](int k) { return static_cast<int8_t*>(P[k]); };
  auto F = [&](int k) { return static_cast<float*>(P[k]); };
  cudaEvent_t* ev_in = h->hp_ev[0];
  cudaEvent_t* ev_y = h->hp_ev[1];
  cudaEvent_t* ev_comp = h->hp_ev[2];
  cudaEvent_t* ev_x = h->hp_ev[4];
  cudaEvent_t* ev_out = h->hp_ev[3];
  cudaStream_t comp = h->stream, s_in = h->s_in, s_out = h->s_out;
  host_pool_begin(h, pi);
  // chunk i covers rows [cuts[i], cuts[i + 1]). Tapered at both ends: a quarter chunk q first, so
  // the first Y leaves (and the D2H direction starts) sooner, and chunks halving down to q at
  // the end, so less compute and fewer bytes (the D2H backlog) are left for the un-overlapped
  // drain after the last upload (9.53 vs 9.58 ms per C2 step with one q chunk last).
  // SB_HOST_FIRST sets q, SB_HOST_TAPER=1 ends with one q chunk, =0 turns the taper off
  // (measurement knobs).
  const char* fe = std::getenv("SB_HOST_FIRST");
  const char* te = std::getenv("SB_HOST_TAPER");
  const bool taper = !(te && te[0] == '0');
  const bool geo = !(te && te[0] == '1');  // end taper: halving toward q (SB_HOST_TAPER=1: one q chunk)
  std::vector<int64_t> cuts{0};
  if (b <= chunk) {  // a batch that fits one chunk stays one chunk
    cuts.push_back(b);
  } else {
    const int64_t q = std::min<int64_t>(chunk, fe ? std::max<int64_t>(128, std::atoll(fe)) : std::max<int64_t>(128, chunk / 4));
    int64_t r = taper ? q : chunk;
    cuts.push_back(r);
    while (r < b) {
      const int64_t rem = b - r;
      const int64_t step = !taper ? std::min(rem, chunk)
                           : geo   ? (rem <= q ? rem : std::min(chunk, std::max(q, rem / 2)))
                           : rem <= q ? rem
                           : rem <= chunk + q ? rem - q
                                              : chunk;
      r += step;
      cuts.push_back(r);
    }
  }
  const int64_t nchunks = static_cast<int64_t>(cuts.size()) - 1;
  auto r0_of = [&](int64_t i) { return cuts[i]; };
  auto rows_of = [&](int64_t i) { return cuts[i + 1] - cuts[i]; };
  // a chunk's x (ev_x: its forward may start) then its g (ev_in: its backward may start)
  auto h2d_x = [&](int64_t i) {
    const int s = static_cast<int>(i % NS);
    const int64_t r0 = r0_of(i), rows = rows_of(i);
    if (i >= NS) cudaStreamWaitEvent(s_in, ev_comp[s], 0);  // slot's x, g consumed by chunk i-NS
    cudaMemcpyAsync(P[NFIX + 4 * s + 0], static_cast<const uint8_t*>(x) + r0 * n * es, rows * n * es,
                    cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev_x[s], s_in);
  };
  auto h2d_g = [&](int64_t i) {
    const int s = static_cast<int>(i % NS);
    const int64_t r0 = r0_of(i), rows = rows_of(i);
    cudaMemcpyAsync(P[NFIX + 4 * s + 1], static_cast<const uint8_t*>(g) + r0 * m * es, rows * m * es,
                    cudaMemcpyHostToDevice, s_in);
    cudaEventRecord(ev_in[s], s_in);
  };
  auto h2d = [&](int64_t i) {
    h2d_x(i);
    h2d_g(i);
  };
  sb_status st = SB_OK;
  // upload order = the order the first chunk's kernels need them: W1, x_0, W2 (the forward),
  // then g_0 (the backward); each weight quantized once (both layouts) as soon as it is in
  cudaMemcpyAsync(P[W1], w1, hd * n * es, cudaMemcpyHostToDevice, s_in);
  cudaEventRecord(h->hp_w1ready, s_in);
  h2d_x(0);
  cudaMemcpyAsync(P[W2], w2, m * hd * es, cudaMemcpyHostToDevice, s_in);
  cudaEventRecord(h->hp_wready, s_in);
  h2d_g(0);
  const char* wl = std::getenv("SB_HOST_W2LATE");
  const bool w2late = !(wl && wl[0] == '0');
  cudaStreamWaitEvent(comp, w2late ? h->hp_w1ready : h->hp_wready, 0);
  st = q_tensorwise(h, P[W1], dt, hd, n, n, I8(W1Q), n, I8(W1QT), hd, F(WST1), static_cast<unsigned int*>(P[WRD1]));
  if (!w2late && st == SB_OK)
    st = q_tensorwise(h, P[W2], dt, m, hd, hd, I8(W2Q), hd, I8(W2QT), m, F(WST2), static_cast<unsigned int*>(P[WRD2]));
  for (int64_t i = 1; i < std::min<int64_t>(NS - 1, nchunks); ++i) h2d(i);
  auto qrow = [&](const void* src, int64_t rows, int64_t cols, int8_t* q, float* s) {
    if (st == SB_OK && sb::launch_quantize_rowwise(h, src, dt, rows, cols, cols, q, cols, s) != cudaSuccess)
      st = sb::cuda_fail(op, cudaGetLastError());
  };
  auto act = [&](int md, const void* a, const void* bb, int64_t rows, void* out, int8_t* q, float* s) {
    if (st == SB_OK && sb::launch_act_quantize_rowwise(h, md, a, bb, rows, hd, out, q, s) != cudaSuccess)
      st = sb::cuda_fail(op, cudaGetLastError());
  };
  for (int64_t i = 0; i < nchunks && st == SB_OK; ++i) {
    const int s = static_cast<int>(i % NS);
    const int64_t r0 = r0_of(i), rows = rows_of(i);
    if (i + NS - 1 < nchunks) h2d(i + NS - 1);
    cudaStreamWaitEvent(comp, ev_x[s], 0);
    if (i >= NS) cudaStreamWaitEvent(comp, ev_out[s], 0);  // slot's y, dx copied out
    void* xd = P[NFIX + 4 * s + 0];
    void* gd = P[NFIX + 4 * s + 1];
    void* yd = P[NFIX + 4 * s + 2];
    void* dxd = P[NFIX + 4 * s + 3];
    // forward
    qrow(xd, rows, n, I8(XQ), F(XS));
    if (st == SB_OK) st = sb::gemm_i8(h, I8(XQ), F(XS), I8(W1Q), F(WST1), SB_SCALE_ROW_TENSOR, rows, hd, n, P[PRE], dt, mode->exact);
    if (gelu)
      act(0, P[PRE], nullptr, rows, P[ACT], I8(HQ), F(HS));
    else
      qrow(P[PRE], rows, hd, I8(HQ), F(HS));
    if (i == 0 && w2late) {  // W2 arrives after x_0: its quantize runs after fc1's first chunk
      cudaStreamWaitEvent(comp, h->hp_wready, 0);
      if (st == SB_OK)
        st = q_tensorwise(h, P[W2], dt, m, hd, hd, I8(W2Q), hd, I8(W2QT), m, F(WST2),
                          static_cast<unsigned int*>(P[WRD2]));
    }
    if (st == SB_OK) st = sb::gemm_i8(h, I8(HQ), F(HS), I8(W2Q), F(WST2), SB_SCALE_ROW_TENSOR, rows, m, hd, yd, dt, mode->exact);
    cudaEventRecord(ev_y[s], comp);
    // backward: fc2 (dW2 with G's quantize in the launch, then dA), then fc1
    cudaStreamWaitEvent(comp, ev_in[s], 0);
    const sb::RowQuant rq2{I8(GQ), m, F(GS)};
    if (st == SB_OK) st = sb::wgrad(h, gd, P[ACT], dt, rows, m, hd, F(DW2), mode->exact, i > 0, &rq2);
    const bool last = i == nchunks - 1;
    // under data parallelism (a communicator on the handle) dW is summed over ranks before it leaves
    if (last && st == SB_OK) st = sb::dp_allreduce_sum_f32(h, F(DW2), m * hd, comp);
    if (last) cudaEventRecord(ev_comp[(s + 1) % NS], comp);  // dW2 complete (that slot's event is not waited on again)
    if (st == SB_OK) st = sb::gemm_i8(h, I8(GQ), F(GS), I8(W2QT), F(WST2), SB_SCALE_ROW_TENSOR, rows, hd, m, P[DA], dt, mode->exact);
    if (gelu) {
      act(1, P[DA], P[PRE], rows, P[G1], I8(G1Q), F(G1S));
      if (st == SB_OK) st = sb::wgrad(h, P[G1], xd, dt, rows, hd, n, F(DW1), mode->exact, i > 0);
    } else {
      const sb::RowQuant rq1{I8(G1Q), hd, F(G1S)};
      if (st == SB_OK) st = sb::wgrad(h, P[G1], xd, dt, rows, hd, n, F(DW1), mode->exact, i > 0, &rq1);
    }
    if (st == SB_OK) st = sb::gemm_i8(h, I8(G1Q), F(G1S), I8(W1QT), F(WST1), SB_SCALE_ROW_TENSOR, rows, n, hd, dxd, dt, mode->exact);
    cudaEventRecord(ev_comp[s], comp);
    cudaStreamWaitEvent(s_out, ev_y[s], 0);
    cudaMemcpyAsync(static_cast<uint8_t*>(y) + r0 * m * es, yd, rows * m * es, cudaMemcpyDeviceToHost, s_out);
    if (last) {  // dW2 leaves while the last chunk's fc1 backward runs
      cudaStreamWaitEvent(s_out, ev_comp[(s + 1) % NS], 0);
      cudaMemcpyAsync(dw2, P[DW2], m * hd * sizeof(float), cudaMemcpyDeviceToHost, s_out);
    }
    cudaStreamWaitEvent(s_out, ev_comp[s], 0);
    cudaMemcpyAsync(static_cast<uint8_t*>(dx) + r0 * n * es, dxd, rows * n * es, cudaMemcpyDeviceToHost, s_out);
    cudaEventRecord(ev_out[s], s_out);
  }
  // as fwd_bwd_host_enqueue: dW1 leaves after the last chunk; the event frees the pool
  if (st == SB_OK) st = sb::dp_allreduce_sum_f32(h, F(DW1), hd * n, comp);
  cudaEventRecord(ev_comp[0], comp);
  cudaStreamWaitEvent(s_out, ev_comp[0], 0);
  cudaMemcpyAsync(dw1, P[DW1], hd * n * sizeof(float), cudaMemcpyDeviceToHost, s_out);
  cudaEventRecord(h->pool_done[pi], s_out);
  h->pool_used[pi] = true;
  return st;
}

}  // extern "C"
namespace {
sb_status host_pipeline_check(sb_handle h, const char* op) {
  cudaError_t e = cudaStreamSynchronize(h->stream);
  cudaStreamSynchronize(h->s_in);
  cudaStreamSynchronize(h->s_out);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return sb::cuda_fail(op, e);
  uint32_t flags = 0;
  cudaMemcpy(&flags, h->d_err, sizeof(flags), cudaMemcpyDeviceToHost);
  if (flags) {
    cudaMemset(h->d_err, 0, sizeof(uint32_t));
    return sb::fail(SB_ERR_NONFINITE, op, "non-finite input");
  }
  return SB_OK;
}
}  // namespace
extern "C" {

sb_status sb_switchback_fwd_bwd_host(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                     const void* g, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y, void* dx,
                                     float* dw) {
  SB_TRY(fwd_bwd_host_enqueue(h, mode, x, w, g, dt, b, n, m, y, dx, dw));
  return host_pipeline_check(h, "switchback_fwd_bwd");
}

sb_status sb_switchback_fwd_bwd_host_async(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                           const void* g, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                                           void* dx, float* dw) {
  return fwd_bwd_host_enqueue(h, mode, x, w, g, dt, b, n, m, y, dx, dw);
}

sb_status sb_switchback_mlp_fwd_bwd_host(sb_handle h, const sb_linear_mode* mode, int activation, const void* x,
                                         const void* w1, const void* w2, const void* g, sb_dtype dt, int64_t b,
                                         int64_t n, int64_t hd, int64_t m, void* y, void* dx, float* dw1, float* dw2) {
  SB_TRY(mlp_host_enqueue(h, mode, activation, x, w1, w2, g, dt, b, n, hd, m, y, dx, dw1, dw2));
  return host_pipeline_check(h, "switchback_mlp_fwd_bwd");
}

sb_status sb_switchback_mlp_fwd_bwd_host_async(sb_handle h, const sb_linear_mode* mode, int activation, const void* x,
                                               const void* w1, const void* w2, const void* g, sb_dtype dt, int64_t b,
                                               int64_t n, int64_t hd, int64_t m, void* y, void* dx, float* dw1,
                                               float* dw2) {
  return mlp_host_enqueue(h, mode, activation, x, w1, w2, g, dt, b, n, hd, m, y, dx, dw1, dw2);
}

sb_status sb_host_pipeline_wait(sb_handle h) {
  SB_TRY(check_h(h, "sb_host_pipeline_wait"));
  if (!h->s_in) return sb_synchronize(h);
  return host_pipeline_check(h, "switchback_fwd_bwd");
}

}  // extern "C"

namespace {
sb_status gemm_bf16(sb_handle h, const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K,
                    void* out, sb_dtype out_dt) {
  float* one = nullptr;
  cudaGetSymbolAddress(reinterpret_cast<void**>(&one), g_one);
  return sb::gemm_bf16_tc(h, a, a_mn, b, b_mn, M, N, K, out, out_dt, one);
}
}  // namespace
