#include <cstdlib>
// util.cu — the remaining C-ABI entries: device memory + copies for FFI callers, the
// device finiteness check (Matrix::all_finite), fp8_cast, the int8 payload transpose, and the
// optimizer helpers compute_rms / grad_clip_global_norm / filter_nonfinite
// (optimizer.cpp:31-42, :72-100). Reductions are fp64 in a fixed tree order (deterministic).
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "sb_internal.h"

namespace {

constexpr int kT = 256;

__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kT / 32; ++i) s = __dadd_rn(s, red[i]);
  __syncthreads();
  return s;
}

template <typename T>
__global__ void k_check_finite(const T* __restrict__ x, int64_t n, uint32_t* err) {
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(static_cast<float>(x[i]));
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

__global__ void k_transpose_i8(const int8_t* __restrict__ in, int64_t rows, int64_t cols, int8_t* __restrict__ out) {
  __shared__ int8_t t[32][33];
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

// partial[b] = sum over this block's slice of f(i); mode 0: g^2/max(u, eps^2), 1: g^2
__global__ void k_partial(const float* __restrict__ g, const float* __restrict__ u, int64_t n, double floor_, int mode,
                          double* __restrict__ partial) {
  __shared__ double red[kT / 32];
  double acc = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = static_cast<int64_t>(blockIdx.x) * per, hi = lo + per < n ? lo + per : n;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kT) {
    const double gi = static_cast<double>(g[i]);
    if (mode == 0) {
      const double ui = static_cast<double>(u[i]);
      acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(gi, gi), ui > floor_ ? ui : floor_));
    } else {
      acc = __dadd_rn(acc, __dmul_rn(gi, gi));
    }
  }
  const double s = block_sum_d(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// out = sqrt(sum(partial) / n) (rms) or the clip factor max/norm (when norm > max) else 1
__global__ void k_finish(const double* __restrict__ partial, int np, double n, int mode, double max_norm, double* out) {
  __shared__ double red[kT / 32];
  double s = 0.0;
  for (int j = threadIdx.x; j < np; j += kT) s = __dadd_rn(s, partial[j]);
  const double tot = block_sum_d(s, red);
  if (threadIdx.x == 0) {
    if (mode == 0) {
      *out = __dsqrt_rn(__ddiv_rn(tot, n));
    } else {
      const double norm = __dsqrt_rn(tot);
      *out = norm > max_norm ? __ddiv_rn(max_norm, norm) : 1.0;
    }
  }
}

__global__ void k_scale(float* __restrict__ g, int64_t n, const double* __restrict__ c) {
  const double cc = *c;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    g[i] = __double2float_rn(__dmul_rn(static_cast<double>(g[i]), cc));
}

__global__ void k_unscale(const float* __restrict__ g, float* __restrict__ o, int64_t n, double scale,
                          int32_t* __restrict__ flag) {
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = __double2float_rn(__ddiv_rn(static_cast<double>(g[i]), scale));
    o[i] = v;
    bad |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(reinterpret_cast<unsigned*>(flag), 1u);
}

// y = float(double(p) * double(s)) == __fmul_rn(p, s) when p is an fp8 value-set member
// (<= 4 significant bits, so the double product is exact); computed in fp64 regardless.
__global__ void k_scale_by_state(const float* __restrict__ p, int64_t rows, int64_t cols, const float* __restrict__ st,
                                 int axis, float* __restrict__ y) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float s = axis == 0 ? st[r] : axis == 1 ? st[c] : st[0];
    y[i] = __double2float_rn(__dmul_rn(static_cast<double>(p[i]), static_cast<double>(s)));
  }
}

__global__ void k_skip_all(int32_t* flags, int n) {
  int any = 0;
  for (int i = 0; i < n; ++i) any |= flags[i];
  if (any)
    for (int i = 0; i < n; ++i) flags[i] = 1;
}

unsigned grid_of(int64_t n, int num_sms) {
  int64_t g = (n + kT * 4 - 1) / (kT * 4);
  if (g > num_sms * 8) g = num_sms * 8;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

sb_status ck(sb_handle h, const char* op) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null handle");
  cudaSetDevice(h->device);
  return SB_OK;
}


// Column sums of a [rows x cols] matrix (leading dim ld) into fp32: the bias gradient of the nn
// module's linears (sum over tokens of G). Block = 8 warps over one strip of 32 * VEC columns
// (16-byte loads, one coalesced 512-byte row segment per warp), rows [r0, r1) of split
// blockIdx.y; warp w takes rows r0 + w, r0 + w + 8, ... (4 loads in flight per thread), the 8
// warps are then summed in order into part[blockIdx.y][...] (or straight into out when there
// is one split), and k_colsum_finish adds the splits in order: deterministic for a given shape.
template <typename T, int VEC>
__global__ void __launch_bounds__(kT) k_colsum(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                                               int64_t rows_per_split, float* __restrict__ part) {
  __shared__ float red[kT / 32][32 * VEC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32 * VEC + lane * VEC;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_split;
  const int64_t r1 = r0 + rows_per_split < rows ? r0 + rows_per_split : rows;
  float acc[VEC];
#pragma unroll
  for (int k = 0; k < VEC; ++k) acc[k] = 0.0f;
  const bool full = c0 + VEC <= cols;
  int64_t r = r0 + w;
  if (VEC > 1 && full) {
    using V = uint4;
    auto add = [&](const V& v) {
      const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] += static_cast<float>(e[k]);
    };
    for (; r + 24 < r1; r += 32) {
      V v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const V*>(x + (r + 8 * u) * ld + c0));
#pragma unroll
      for (int u = 0; u < 4; ++u) add(v[u]);
    }
    for (; r < r1; r += 8) add(__ldg(reinterpret_cast<const V*>(x + r * ld + c0)));
  } else {
    for (; r < r1; r += 8)
#pragma unroll
      for (int k = 0; k < VEC; ++k)
        if (c0 + k < cols) acc[k] += static_cast<float>(x[r * ld + c0 + k]);
  }
#pragma unroll
  for (int k = 0; k < VEC; ++k) red[w][lane * VEC + k] = acc[k];
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * VEC; t += kT) {
    const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 * VEC + t;
    if (c >= cols) continue;
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < kT / 32; ++i) s += red[i][t];
    part[static_cast<int64_t>(blockIdx.y) * cols + c] = s;
  }
}

// out[c] = sum over splits of part[i][c]: block = 32 columns x 8 warps, warp w adds splits
// w, w + 8, ... (coalesced 128-byte rows), then the 8 warp sums in order.
__global__ void __launch_bounds__(kT) k_colsum_finish(const float* __restrict__ part, int splits, int64_t cols,
                                                      float* __restrict__ out) {
  __shared__ float red[kT / 32][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  float s = 0.0f;
  if (c < cols)
    for (int i = w; i < splits; i += kT / 32) s += part[static_cast<int64_t>(i) * cols + c];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = 0.0f;
#pragma unroll
    for (int i = 0; i < kT / 32; ++i) t += red[i][lane];
    out[c] = t;
  }
}

template <typename T>
sb_status colsum_launch(sb_handle h, const T* x, int64_t rows, int64_t cols, int64_t ld, float* out) {
  constexpr int VEC = 16 / sizeof(T);
  const bool vec = cols % VEC == 0 && ld % VEC == 0 && sb::aligned(x, 16);
  const int per = vec ? 32 * VEC : 32;
  const int64_t strips = (cols + per - 1) / per;
  // ~8 resident blocks per SM; the split partials live in the stream's scratch (<= 1 MB, the
  // capture-time buffer's size)
  int64_t splits = (static_cast<int64_t>(h->num_sms) * 8 + strips - 1) / strips;
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, rows / 64));
  splits = std::min<int64_t>(splits, std::max<int64_t>(1, (1 << 20) / (cols * 4)));
  splits = std::max<int64_t>(splits, 1);
  const int64_t rps = (rows + splits - 1) / splits;
  splits = (rows + rps - 1) / rps;
  float* part = out;
  if (splits > 1) {
    part = reinterpret_cast<float*>(sb::scratch(h, static_cast<size_t>(splits * cols)));
    if (!part) return sb::fail(SB_ERR_CUDA, "column_sums", "scratch allocation failed (or would grow inside a graph capture: run the op once on this stream first)");
  }
  const dim3 grid(static_cast<unsigned>(strips), static_cast<unsigned>(splits));
  h->launches++;
  if (vec)
    k_colsum<T, VEC><<<grid, kT, 0, h->stream>>>(x, rows, cols, ld, rps, part);
  else
    k_colsum<T, 1><<<grid, kT, 0, h->stream>>>(x, rows, cols, ld, rps, part);
  if (splits > 1) {
    h->launches++;
    k_colsum_finish<<<static_cast<unsigned>((cols + 31) / 32), kT, 0, h->stream>>>(part, static_cast<int>(splits), cols,
                                                                                   out);
  }
  SB_LAUNCH_CHECK("column_sums");
  return SB_OK;
}

}  // namespace

extern "C" {

sb_status sb_device_alloc(sb_handle h, size_t bytes, void** out) {
  if (ck(h, "sb_device_alloc") != SB_OK || !out) return SB_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  if (bytes == 0) return SB_OK;
  SB_CUDA_CHECK("sb_device_alloc", cudaMalloc(out, bytes));
  return SB_OK;
}

sb_status sb_device_free(sb_handle h, void* p) {
  if (ck(h, "sb_device_free") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (p) {
    cudaStreamSynchronize(h->stream);
    SB_CUDA_CHECK("sb_device_free", cudaFree(p));
  }
  return SB_OK;
}

sb_status sb_copy_to_device(sb_handle h, void* dst, const void* src, size_t bytes) {
  if (ck(h, "sb_copy_to_device") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (!bytes) return SB_OK;
  SB_CUDA_CHECK("sb_copy_to_device", cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, h->stream));
  SB_CUDA_CHECK("sb_copy_to_device", cudaStreamSynchronize(h->stream));
  return SB_OK;
}

sb_status sb_copy_to_host(sb_handle h, void* dst, const void* src, size_t bytes) {
  if (ck(h, "sb_copy_to_host") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (!bytes) return SB_OK;
  SB_CUDA_CHECK("sb_copy_to_host", cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, h->stream));
  SB_CUDA_CHECK("sb_copy_to_host", cudaStreamSynchronize(h->stream));
  return SB_OK;
}

sb_status sb_check_finite(sb_handle h, const void* x, sb_dtype dt, int64_t n) {
  if (ck(h, "all_finite") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (n <= 0) return SB_OK;
  h->launches++;
  if (dt == SB_BF16)
    k_check_finite<<<grid_of(n, h->num_sms), kT, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), n, h->d_err);
  else if (dt == SB_F32)
    k_check_finite<<<grid_of(n, h->num_sms), kT, 0, h->stream>>>(static_cast<const float*>(x), n, h->d_err);
  else
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "all_finite", "float input expected");
  SB_LAUNCH_CHECK("all_finite");
  return SB_OK;
}

sb_status sb_fp8_cast(sb_handle h, const float* x, int64_t n, sb_fp8_format fmt, float* y) {
  if (ck(h, "fp8_cast") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (fmt != SB_E4M3 && fmt != SB_E5M2) return sb::fail(SB_ERR_UNSUPPORTED, "fp8_cast", "only e4m3 / e5m2 on device");
  if (n <= 0) return SB_OK;
  SB_CUDA_CHECK("fp8_cast", sb::launch_fp8_cast(h, x, n, fmt, y));
  return SB_OK;
}

sb_status sb_dequantize_values(sb_handle h, const float* p, int64_t rows, int64_t cols, const float* state, sb_axis axis,
                               float* y) {
  if (ck(h, "dequantize") != SB_OK || !p || !state || !y || axis < 0 || axis > 2)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "dequantize", "state length does not match axis");
  if (rows <= 0 || cols <= 0) return SB_OK;
  h->launches++;
  k_scale_by_state<<<grid_of(rows * cols, h->num_sms), kT, 0, h->stream>>>(p, rows, cols, state, axis, y);
  SB_LAUNCH_CHECK("dequantize");
  return SB_OK;
}

sb_status sb_transpose_i8(sb_handle h, const int8_t* in, int64_t rows, int64_t cols, int8_t* out) {
  if (ck(h, "transpose") != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (rows <= 0 || cols <= 0) return SB_OK;
  h->launches++;
  k_transpose_i8<<<dim3(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32)), dim3(32, 8), 0,
                   h->stream>>>(in, rows, cols, out);
  SB_LAUNCH_CHECK("transpose");
  return SB_OK;
}

sb_status sb_column_sums(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ld, float* out) {
  const char* op = "column_sums";
  if (ck(h, op) != SB_OK || (!x && rows > 0) || !out || cols <= 0 || rows < 0 || ld < cols || (dt != SB_BF16 && dt != SB_F32))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (bf16 / fp32, ld >= cols > 0)");
  if (rows == 0) {
    cudaMemsetAsync(out, 0, static_cast<size_t>(cols) * sizeof(float), h->stream);
    SB_LAUNCH_CHECK(op);
    return SB_OK;
  }
  return dt == SB_BF16 ? colsum_launch(h, static_cast<const __nv_bfloat16*>(x), rows, cols, ld, out)
                       : colsum_launch(h, static_cast<const float*>(x), rows, cols, ld, out);
}

sb_status sb_compute_rms(sb_handle h, const float* g, const float* u, int64_t n, double eps, double* out) {
  const char* op = "compute_rms";
  if (ck(h, op) != SB_OK || !g || !u || !out) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "shape mismatch");
  if (n <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "empty input");
  const int np = static_cast<int>(grid_of(n, h->num_sms));
  double* partial = reinterpret_cast<double*>(sb::scratch(h, 2 * static_cast<size_t>(np) + 2));
  if (!partial) return sb::fail(SB_ERR_CUDA, op, "scratch allocation failed (or would grow inside a graph capture: run the op once on this stream first)");
  h->launches += 2;
  k_partial<<<np, kT, 0, h->stream>>>(g, u, n, eps * eps, 0, partial);
  k_finish<<<1, kT, 0, h->stream>>>(partial, np, static_cast<double>(n), 0, 0.0, out);
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

sb_status sb_grad_clip_global_norm(sb_handle h, float* const* grads, const int64_t* numel, int n, double max_norm) {
  const char* op = "grad_clip";
  if (ck(h, op) != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (!(max_norm > 0)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "max_norm must be > 0");  // optimizer.cpp:73
  if (n <= 0) return SB_OK;
  std::vector<int> np(static_cast<size_t>(n));
  int total = 0;
  for (int i = 0; i < n; ++i) {
    np[static_cast<size_t>(i)] = numel[i] > 0 ? static_cast<int>(grid_of(numel[i], h->num_sms)) : 0;
    total += np[static_cast<size_t>(i)];
  }
  double* partial = reinterpret_cast<double*>(sb::scratch(h, 2 * static_cast<size_t>(total) + 4));
  if (!partial) return sb::fail(SB_ERR_CUDA, op, "scratch allocation failed (or would grow inside a graph capture: run the op once on this stream first)");
  double* clip = partial + total;
  int off = 0;
  for (int i = 0; i < n; ++i) {
    if (!np[static_cast<size_t>(i)]) continue;
    h->launches++;
    k_partial<<<np[static_cast<size_t>(i)], kT, 0, h->stream>>>(grads[i], nullptr, numel[i], 0.0, 1, partial + off);
    off += np[static_cast<size_t>(i)];
  }
  h->launches++;
  k_finish<<<1, kT, 0, h->stream>>>(partial, total, 0.0, 1, max_norm, clip);
  for (int i = 0; i < n; ++i) {
    if (numel[i] <= 0) continue;
    h->launches++;
    k_scale<<<grid_of(numel[i], h->num_sms), kT, 0, h->stream>>>(grads[i], numel[i], clip);
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

sb_status sb_filter_nonfinite(sb_handle h, const float* const* grads, float* const* out, const int64_t* numel, int n,
                              double scale, int per_tensor_skip, int32_t* skipped) {
  const char* op = "loss scaler";
  if (ck(h, op) != SB_OK) return SB_ERR_INVALID_ARGUMENT;
  if (!(scale > 0)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "scale must be > 0");  // optimizer.cpp:84
  if (n <= 0) return SB_OK;
  SB_CUDA_CHECK(op, cudaMemsetAsync(skipped, 0, sizeof(int32_t) * n, h->stream));
  for (int i = 0; i < n; ++i) {
    if (numel[i] <= 0) continue;
    h->launches++;
    k_unscale<<<grid_of(numel[i], h->num_sms), kT, 0, h->stream>>>(grads[i], out[i], numel[i], scale, skipped + i);
  }
  if (!per_tensor_skip) {
    h->launches++;
    k_skip_all<<<1, 1, 0, h->stream>>>(skipped, n);
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

}  // extern "C"

namespace sb {
bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SB_PDL");
    v = (e && e[0] == '1') ? 1 : 0;  // default off: measured 1% slower on the C2 step
  }
  return v == 1;
}
}  // namespace sb
