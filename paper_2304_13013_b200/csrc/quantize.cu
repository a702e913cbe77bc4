// quantize.cu — HBM-bound quantize / dequantize kernels of the SwitchBack path.
//
//   K1 quantize_rowwise           quantize.cpp:116-133 (slice_absmax :89-112, quantize_entry :17-20)
//   K2 tensor absmax              Matrix::abs_max, matrix.cpp:32-36
//   K3 tensor-wise quantize (+ transposed copy in the same pass)   quantize.cpp:139-159
//   K4 column-wise absmax / quantize (+ transposed = rowwise(W^T)) quantize.cpp:135-137, linear.cpp:228-229
//   K8 fp8 quantize, ties to the smaller magnitude               quantize.cpp:65-76,161-176
//   K10 dequantize (int8 / fp8)                                  quantize.cpp:178-197
//
// Bit-exactness of the int8 payload. The reference computes
// lround(127.0*double(x)/double(s)). Because |127x/s - (k+1/2)| >= 2^-33 whenever it is
// not an exact tie (x, s floats), the double quotient never moves a rounding
// decision, so the payload is round-half-away-from-zero of the EXACT rational
// 127|x|/s. We take a fast fp32 candidate k = floor(127|x|*(127/s)^-... + 1/2) and then
// decide exactly between k-1, k, k+1 by comparing 127|x| with (k +- 1/2)*s:
//   bf16 input: both products are exact in fp32 (<= 16 significant bits),
//   fp32 input: the comparison runs in fp64 (31- and 33-bit products, exact) but only
//               when the candidate is within 1e-3 of a half-integer.
// Rows with tiny / huge absmax are pre-scaled by an exact power of two.
//
// Absmax uses an integer max over the sign-cleared bit patterns: for non-negative
// floats integer order == float order, and NaN/Inf (>= 0x7f800000) surface as the
// maximum, which is how non-finite input is detected (fmaxf would drop NaN).
#include <cuda_bf16.h>

#include <algorithm>
#include <type_traits>

#include "sb_internal.h"
#include "sb_ptx.cuh"
#include "quant_core.cuh"

namespace {

using namespace sbq;

// ------------------------------------------------------------------ K1 ----
// TMA-fed row-wise quantizer. One producer lane streams whole rows of X with
// cp.async.bulk (16-byte aligned rows) into a ring of smem slots (mbarrier full/empty
// pairs); 8 consumer warps each own every 8th row of the block's share: absmax over the
// row from smem (integer max of |x| bit patterns), then the quantize pass from smem, int8
// payload written with coalesced 8-/4-byte stores. HBM sees one read of X and one write of
// the payload; the ring keeps ~100 KB of reads in flight per block (2 blocks per SM).
constexpr int kQWarps = 12;                    // consumer warps per block (2 blocks / SM)
constexpr int kQThreads = 32 * (kQWarps + 1);  // + 1 producer warp
constexpr int kQRingBytes = 100 * 1024;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sbptx::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sbptx::smem_u32(bar))
               : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kQThreads) k_quantize_rowwise_tma(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                                   int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                   float* __restrict__ state, uint32_t* err,
                                                                   int stages, int slot_bytes) {
  constexpr int VEC = 16 / sizeof(T);
  using Out = typename VecQ<T>::Out;
  extern __shared__ __align__(128) uint8_t qsmem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(qsmem + static_cast<size_t>(stages) * slot_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = static_cast<uint32_t>(cols * sizeof(T));
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      sbptx::mbar_init(&full[s], 1);
      sbptx::mbar_init(&empty[s], 1);
    }
    sbptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == kQWarps) {
    if (lane == 0) {  // producer
      int i = 0;
      for (int64_t row = blockIdx.x; row < rows; row += gridDim.x, ++i) {
        const int s = i % stages;
        const uint32_t ph = static_cast<uint32_t>(i / stages) & 1u;
        sbptx::mbar_wait(&empty[s], ph ^ 1u);
        sbptx::mbar_arrive_expect_tx(&full[s], row_bytes);
        bulk_load(qsmem + static_cast<size_t>(s) * slot_bytes, x + row * ldx, row_bytes, &full[s]);
      }
    }
    return;
  }
  const int nvec = static_cast<int>(cols / VEC);
  // A consumer must never wait on a slot more than one phase ahead (try_wait.parity on the
  // previous parity returns at once). The launcher makes `stages` a multiple of the active
  // consumer count, so slot s only ever holds rows of consumer s % active: each consumer
  // waits on its own slots' phases in order, having consumed the previous phase itself.
  const int active = kQWarps < stages ? kQWarps : stages;
  if (warp >= active) return;
  int i = warp;
  for (int64_t row = blockIdx.x + static_cast<int64_t>(warp) * gridDim.x; row < rows;
       row += static_cast<int64_t>(active) * gridDim.x, i += active) {
    const int s = i % stages;
    const uint32_t ph = static_cast<uint32_t>(i / stages) & 1u;
    sbptx::mbar_wait(&full[s], ph);
    const uint4* xs = reinterpret_cast<const uint4*>(qsmem + static_cast<size_t>(s) * slot_bytes);
    uint32_t amax = 0;
#pragma unroll 4
    for (int v = lane; v < nvec; v += 32) amax = max(amax, vec_absmax_bits<T>(xs[v]));
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        state[row] = __uint_as_float(amax);
      }
    } else {
      const float st = state_from_bits(amax);
      if (lane == 0) state[row] = st;
      const Scale sc = make_scale(st);
      const bool plain = sc.pre == 1.0f;
      Out* qr = reinterpret_cast<Out*>(q + row * ldq);
      // warp-uniform trip count: qvec() votes across the warp (__any_sync)
#pragma unroll 4
      for (int b = 0; b < nvec; b += 32) {
        const int v = b + lane;
        const Out o = qvec<T>(v < nvec ? xs[v] : make_uint4(0, 0, 0, 0), sc, plain);
        if (v < nvec) qr[v] = o;
      }
    }
    __syncwarp();
    if (lane == 0) sbptx::mbar_arrive(&empty[s]);
  }
}

// Rows longer than a ring slot: one warp per row, second pass re-reads (L2 hit).
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_rowwise_stream(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                                  int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                  float* __restrict__ state, uint32_t* err) {
  constexpr int VEC = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  quantize_row_stream<T>(reinterpret_cast<const uint4*>(x + row * ldx), cols / VEC, q + row * ldq, state + row, err,
                         lane);
}

// Any shape / alignment: scalar element access.
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_rowwise_scalar(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                                  int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                  float* __restrict__ state, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * ldx;
  uint32_t amax = 0;
  for (int64_t j = lane; j < cols; j += 32) amax = max(amax, abs_bits<T>(xr[j]));
  amax = __reduce_max_sync(0xffffffffu, amax);
  if (amax >= kNonFiniteBits) {
    if (lane == 0) {
      raise_nonfinite(err);
      state[row] = __uint_as_float(amax);
    }
    return;
  }
  const float s = state_from_bits(amax);
  if (lane == 0) state[row] = s;
  const Scale sc = make_scale(s);
  for (int64_t j = lane; j < cols; j += 32) q[row * ldq + j] = quantize_one(xr[j], sc);
}

// Register-resident row-wise quantizer: one warp owns a whole row (up to 32*VPL 16-byte
// vectors). All of the row's loads are issued before the first use (VPL independent 16-byte
// loads per lane in flight), the absmax is a warp reduction, and the payload is produced from
// the same registers — one HBM read of X, one write of the payload, no shared memory. Enough
// warps per SM stay resident (launch bounds) to keep ~100+ KB of reads in flight per SM.
template <typename T, int VPL>
__global__ void __launch_bounds__(256) k_quantize_rowwise_reg(const T* __restrict__ x, int64_t rows, int nvec,
                                                              int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                              float* __restrict__ state, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  sbptx::pdl_trigger();
  sbptx::pdl_wait();
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps)
    quantize_row_reg<T, VPL>(reinterpret_cast<const uint4*>(x + row * ldx), nvec, q + row * ldq, state + row, err, lane);
}

template <typename T, int VPL>
void launch_reg(sb_handle h, const T* x, int64_t rows, int nvec, int64_t ldx, int8_t* q, int64_t ldq, float* state) {
  static int blocks_per_sm = 0;
  if (blocks_per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_quantize_rowwise_reg<T, VPL>, 256, 0) !=
            cudaSuccess ||
        blocks_per_sm < 1)
      blocks_per_sm = 1;
  }
  const int64_t need = (rows + 7) / 8;
  const int64_t blocks = std::min<int64_t>(need, static_cast<int64_t>(h->num_sms) * blocks_per_sm);
  sb::launch_pdl(k_quantize_rowwise_reg<T, VPL>, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, h->stream, x, rows,
                 nvec, ldx, q, ldq, state, h->d_err);
}

// Dispatch on vectors-per-lane; false when the row is too long for registers.
template <typename T>
bool rowwise_reg(sb_handle h, const T* x, int64_t rows, int nvec, int64_t ldx, int8_t* q, int64_t ldq, float* state) {
  const int vpl = (nvec + 31) / 32;
  switch (vpl) {
    case 1: launch_reg<T, 1>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 2: launch_reg<T, 2>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 3: launch_reg<T, 3>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 4: launch_reg<T, 4>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 5: launch_reg<T, 5>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 6: launch_reg<T, 6>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 7:
    case 8: launch_reg<T, 8>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 9:
    case 10: launch_reg<T, 10>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 11:
    case 12: launch_reg<T, 12>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 13:
    case 14:
    case 15:
    case 16: launch_reg<T, 16>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 17:
    case 18:
    case 19:
    case 20: launch_reg<T, 20>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    case 21:
    case 22:
    case 23:
    case 24: launch_reg<T, 24>(h, x, rows, nvec, ldx, q, ldq, state); return true;
    default: return false;
  }
}

// ---- producer fusion: activation + row-wise quantize -------------
// The MLP's GELU (forward) and GELU backward produce exactly the rows the next SwitchBack
// GEMM quantizes row-wise. One kernel computes the activation row into registers, stores
// it (bf16: the weight gradient needs it), and quantizes the SAME register values: one read
// of the producer's input instead of write + re-read. The payload and states are those of
// quantize_rowwise(act) bit for bit (identical qvec / state path on identical bf16 values).
//   MODE 0: act = gelu(a)            (erf form, as torch.nn.functional.gelu)
//   MODE 1: act = a * gelu'(b)       (a = upstream gradient, b = the GELU input)
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752440f));
}
__device__ __forceinline__ float gelu_grad_f(float dy, float x) {
  const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752440f));
  const float pdf = expf(-0.5f * x * x) * 0.39894228040143267794f;
  return dy * (cdf + x * pdf);
}
// bf16 inputs take only 65536 values, so GELU and GELU' are tabulated once per handle with
// the formulas above (build_gelu_lut) and read from shared memory: a lookup instead of ~40
// instructions of erf/exp per element, bit-identical to the formula (the table IS the
// formula's output; tests/test_nn_gpu.py checks every bf16 input).
//   forward: all 65536 bf16 results (128 KB), indexed by the raw bits -- no range test.
//   backward: the fp32 factor cdf + x*pdf for |x| < 16 (131 KB; a full fp32 table would not
//   fit). Beyond it the formula saturates exactly in fp32: erf(+-x/sqrt2) = +-1 and
//   exp(-x^2/2) underflows to 0, so the factor is 1 (x >= 16), +0 (x <= -16), NaN (inf/NaN:
//   inf * 0): a select, no divergent branch.
constexpr uint32_t kLutHalf = 0x4180u;  // bf16 bits of 16.0: |x| < 16 <=> (bits & 0x7fff) < kLutHalf
constexpr int kLutEntries = 2 * kLutHalf;
constexpr int kFwdEntries = 65536;
__global__ void k_build_gelu_lut(__nv_bfloat16* fwd, float* grad_factor) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kFwdEntries; i += gridDim.x * blockDim.x) {
    const float x = __bfloat162float(__ushort_as_bfloat16(static_cast<unsigned short>(i)));
    fwd[i] = __float2bfloat16_rn(gelu_f(x));
    if (i < kLutEntries) {
      const uint32_t bits = i < static_cast<int>(kLutHalf) ? static_cast<uint32_t>(i) : 0x8000u + (i - kLutHalf);
      const float xb = __bfloat162float(__ushort_as_bfloat16(static_cast<unsigned short>(bits)));
      const float cdf = 0.5f * (1.0f + erff(xb * 0.70710678118654752440f));
      const float pdf = expf(-0.5f * xb * xb) * 0.39894228040143267794f;
      grad_factor[i] = cdf + xb * pdf;  // gelu_grad_f(dy, x) == dy * grad_factor (same ops, no fma)
    }
  }
}
__device__ __forceinline__ float gelu_grad_factor(uint32_t xb, const float* lut) {
  const uint32_t mag = xb & 0x7fffu;
  const uint32_t neg = xb >> 15;
  const bool in = mag < kLutHalf;
  const float t = lut[in ? neg * kLutHalf + mag : 0u];
  const float sat = mag >= 0x7f80u ? __int_as_float(0x7fffffff) : (neg ? 0.0f : 1.0f);
  return in ? t : sat;
}

template <int MODE>
__device__ __forceinline__ uint4 act_vec(const uint4& a, const uint4& b, const void* lut) {
  uint4 r;
  const uint32_t* wa = reinterpret_cast<const uint32_t*>(&a);
  const uint32_t* wb = reinterpret_cast<const uint32_t*>(&b);
  uint32_t* wr = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    uint32_t out = 0;
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      const uint32_t xa = (wa[k] >> (16 * hf)) & 0xffffu;  // MODE 0: x; MODE 1: dy
      uint32_t o;
      if (MODE == 0) {
        o = static_cast<const unsigned short*>(lut)[xa];
      } else {
        const uint32_t xb = (wb[k] >> (16 * hf)) & 0xffffu;  // x
        const float dy = __bfloat162float(__ushort_as_bfloat16(static_cast<unsigned short>(xa)));
        const float gv = dy * gelu_grad_factor(xb, static_cast<const float*>(lut));
        o = __bfloat16_as_ushort(__float2bfloat16_rn(gv));
      }
      out |= o << (16 * hf);
    }
    wr[k] = out;
  }
  return r;
}

// One warp per row, in chunks of 4 vectors per lane: pass 1 computes the activation, stores
// it and takes the absmax; pass 2 re-reads the just-written row (an L2 hit) and quantizes.
// The GELU math is long (erf, exp), so the row is NOT held in registers across it: a
// register-resident row (the plain quantizer's design) needs ~210 registers here and runs
// 2-3x slower at 12% occupancy.
constexpr int kActThreads = 1024;
template <int MODE, int CH>
__global__ void __launch_bounds__(kActThreads, 1) k_act_quantize_rows(const __nv_bfloat16* __restrict__ a,
                                                                     const __nv_bfloat16* __restrict__ b, int64_t rows,
                                                                     int nvec, __nv_bfloat16* __restrict__ act,
                                                                     int8_t* __restrict__ q, float* __restrict__ state,
                                                                     uint32_t* err, const uint4* __restrict__ lut_g) {
  using T = __nv_bfloat16;
  using Out = typename VecQ<T>::Out;
  constexpr int LUT_VECS = (MODE == 0 ? kFwdEntries * 2 : kLutEntries * 4) / 16;
  extern __shared__ uint4 lut_s[];
  for (int i = threadIdx.x; i < LUT_VECS; i += blockDim.x) lut_s[i] = __ldg(lut_g + i);
  __syncthreads();
  const void* lut = lut_s;
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const int64_t off = row * static_cast<int64_t>(nvec);
    const uint4* ar = reinterpret_cast<const uint4*>(a) + off;
    const uint4* br = reinterpret_cast<const uint4*>(b) + off;
    uint4* outr = reinterpret_cast<uint4*>(act) + off;
    uint32_t amax = 0;
    for (int c0 = 0; c0 < nvec; c0 += 32 * CH) {
      uint4 v[CH], w[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int i = c0 + j * 32 + lane;
        v[j] = i < nvec ? ld_stream(ar + i) : make_uint4(0, 0, 0, 0);
        if (MODE == 1) w[j] = i < nvec ? ld_stream(br + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int i = c0 + j * 32 + lane;
        const uint4 r = act_vec<MODE>(v[j], MODE == 1 ? w[j] : v[j], lut);
        if (i < nvec) {
          outr[i] = r;
          amax = max(amax, vec_absmax_bits<T>(r));
        }
      }
    }
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        state[row] = __uint_as_float(amax);
      }
      continue;
    }
    const float st = state_from_bits(amax);
    if (lane == 0) state[row] = st;
    const Scale sc = make_scale(st);
    const bool plain = sc.pre == 1.0f;
    __syncwarp();  // this warp's act stores precede its re-reads
    Out* qr = reinterpret_cast<Out*>(q + off * 8);
    for (int c0 = 0; c0 < nvec; c0 += 32 * CH) {  // warp-uniform trip count (qvec votes)
      uint4 v[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int i = c0 + j * 32 + lane;
        v[j] = i < nvec ? __ldcg(outr + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int i = c0 + j * 32 + lane;
        const Out o = qvec<T>(v[j], sc, plain);
        if (i < nvec) qr[i] = o;
      }
    }
  }
}

// Any shape: the activation elementwise (same formulas), then the row-wise quantizer.
template <int MODE>
__global__ void k_act_elementwise(const __nv_bfloat16* __restrict__ a, const __nv_bfloat16* __restrict__ b, int64_t n,
                                  __nv_bfloat16* __restrict__ act) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float x = __bfloat162float(a[i]);
    act[i] = __float2bfloat16_rn(MODE == 0 ? gelu_f(x) : gelu_grad_f(x, __bfloat162float(b[i])));
  }
}

template <int MODE, int CH>
cudaError_t launch_act_rows(sb_handle h, const __nv_bfloat16* a, const __nv_bfloat16* b, int64_t rows, int nvec,
                            __nv_bfloat16* act, int8_t* q, float* state) {
  const size_t smem = MODE == 0 ? static_cast<size_t>(kFwdEntries) * 2 : static_cast<size_t>(kLutEntries) * 4;
  static bool attr[16] = {};  // the smem attribute is per device context
  if (!attr[h->device & 15]) {
    const cudaError_t e = cudaFuncSetAttribute(k_act_quantize_rows<MODE, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr[h->device & 15] = true;
  }
  const uint4* lut = reinterpret_cast<const uint4*>(static_cast<const uint8_t*>(h->gelu_lut) +
                                                    (MODE == 0 ? 0 : static_cast<size_t>(kFwdEntries) * 2));
  const int64_t need = (rows + 31) / 32;
  const int64_t blocks = std::min<int64_t>(need, static_cast<int64_t>(h->num_sms));
  h->launches++;
  k_act_quantize_rows<MODE, CH><<<static_cast<unsigned>(blocks), kActThreads, smem, h->stream>>>(a, b, rows, nvec, act,
                                                                                                 q, state, h->d_err, lut);
  return cudaGetLastError();
}

// ---- producer fusion: LayerNorm + row-wise quantize -----------------
// A pre-norm block feeds LayerNorm(x) straight into a SwitchBack linear. One warp per row,
// the row in registers: mean and variance (two passes over the registers, fp32), the affine
// output rounded to bf16 and stored (the dW GEMM needs it), then the same register values
// quantized row-wise; mean / rstd are written for the backward. Payload / states equal
// quantize_rowwise(h) bit for bit.
template <int VPL>
__device__ __forceinline__ void ln_row(uint4 (&v)[VPL], int64_t row, int nvec, int lane, float inv_n, float eps,
                                       const float4* gb_s, __nv_bfloat16* __restrict__ h, int8_t* __restrict__ q,
                                       float* __restrict__ state, float* __restrict__ mean_out,
                                       float* __restrict__ rstd_out, uint32_t* err) {
  using T = __nv_bfloat16;
  using Out = typename VecQ<T>::Out;
  const int64_t off = row * static_cast<int64_t>(nvec);
  // the element math runs on the packed fp32x2 pipe (FADD2 / FFMA2 / FMUL2): two columns per
  // instruction, half the issue slots of the scalar form
  float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[j]);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc = __fadd2_rn(acc, __bfloat1622float2(p2[k]));
  }
  float sum = acc.x + acc.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const float mean = sum * inv_n;
  const float2 nmean = make_float2(-mean, -mean);
  float2 acc2 = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    if (j * 32 + lane >= nvec) continue;
    const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&v[j]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 d = __fadd2_rn(__bfloat1622float2(p2[k]), nmean);
      acc2 = __ffma2_rn(d, d, acc2);
    }
  }
  float sq = acc2.x + acc2.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    const float rstd = rsqrtf(sq * inv_n + eps);
    const float2 rs2 = make_float2(rstd, rstd);
    uint4* hr = reinterpret_cast<uint4*>(h) + off;
    uint32_t amax = 0;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = j * 32 + lane;
      if (i >= nvec) continue;
      const float4 g0 = gb_s[2 * i], g1 = gb_s[2 * i + 1];
      const float4 b0 = gb_s[2 * 32 * VPL + 2 * i], b1 = gb_s[2 * 32 * VPL + 2 * i + 1];
      const float2 gg[4] = {make_float2(g0.x, g0.y), make_float2(g0.z, g0.w), make_float2(g1.x, g1.y),
                            make_float2(g1.z, g1.w)};
      const float2 bb[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                            make_float2(b1.z, b1.w)};
      __nv_bfloat162* p2 = reinterpret_cast<__nv_bfloat162*>(&v[j]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 xh = __fmul2_rn(__fadd2_rn(__bfloat1622float2(p2[k]), nmean), rs2);
        p2[k] = __float22bfloat162_rn(__ffma2_rn(xh, gg[k], bb[k]));
      }
      hr[i] = v[j];
      amax = max(amax, vec_absmax_bits<T>(v[j]));
    }
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (lane == 0) {
      mean_out[row] = mean;
      rstd_out[row] = rstd;
    }
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        state[row] = __uint_as_float(amax);
      }
      return;
    }
    const float st = state_from_bits(amax);
    if (lane == 0) state[row] = st;
    const Scale sc = make_scale(st);
    const bool plain = sc.pre == 1.0f;
    Out* qr = reinterpret_cast<Out*>(q + off * 8);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      if (j * 32 >= nvec) break;  // warp-uniform (qvec votes across the warp)
      const int i = j * 32 + lane;
      const Out o = qvec<T>(v[j], sc, plain);
      if (i < nvec) qr[i] = o;
    }
}

// ---- producer fusion: attention gradients -> the q/k/v projection's packed G + its quantize --
// The grouped q/k/v linear (three projections of one input, model.cpp:303-305) gets its output
// gradients from attention as three head-major tensors dq, dk, dv [B, H, S, Dh] (any strides, Dh
// contiguous). One warp per (token row t = b S + s, projection i): gather the row's H x Dh values
// (the layout change a torch caller does with three strided copies), write them into the packed
// G [T x 3D] the dW GEMM reads, and quantize them row-wise from the same registers into the
// projection's payload q_i [T x D] / states s_i [T] — equal to quantize_rowwise(G[:, iD:(i+1)D]).
struct HeadsSrc {
  const __nv_bfloat16* p[3];
  int64_t sb[3], sh[3], ss[3];  // element strides of b, h, s (Dh stride 1)
  int8_t* q[3];
  float* st[3];
};

template <int VPL>
__global__ void __launch_bounds__(256) k_heads_pack_quantize(const __grid_constant__ HeadsSrc src, int64_t S, int H,
                                                             int Dh, int64_t T, __nv_bfloat16* __restrict__ g,
                                                             uint32_t* err) {
  using T16 = __nv_bfloat16;
  using Out = typename VecQ<T16>::Out;
  const int lane = threadIdx.x & 31;
  const int D = H * Dh, nvec = D / 8, vph = Dh / 8;  // 16-byte vectors per row / per head
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); w < 3 * T; w += warps) {
    const int i = static_cast<int>(w % 3);
    const int64_t t = w / 3, b = t / S, s = t - b * S;
    const T16* base = src.p[i] + b * src.sb[i] + s * src.ss[i];
    uint4 v[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int k = j * 32 + lane;
      if (k < nvec) {
        const int hh = k / vph, wi = k - hh * vph;
        v[j] = ld_stream(reinterpret_cast<const uint4*>(base + hh * src.sh[i] + wi * 8));
      } else {
        v[j] = make_uint4(0, 0, 0, 0);
      }
    }
    uint4* grow = reinterpret_cast<uint4*>(g + t * 3 * D + i * D);
    uint32_t amax = 0;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int k = j * 32 + lane;
      if (k < nvec) grow[k] = v[j];
      amax = max(amax, vec_absmax_bits<T16>(v[j]));
    }
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        src.st[i][t] = __uint_as_float(amax);
      }
      continue;
    }
    const float stv = state_from_bits(amax);
    if (lane == 0) src.st[i][t] = stv;
    const Scale sc = make_scale(stv);
    const bool plain = sc.pre == 1.0f;
    Out* qr = reinterpret_cast<Out*>(src.q[i] + t * D);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      if (j * 32 >= nvec) break;  // warp-uniform (qvec votes across the warp)
      const int k = j * 32 + lane;
      const Out o = qvec<T16>(v[j], sc, plain);
      if (k < nvec) qr[k] = o;
    }
  }
}

// NR rows per warp step: all NR rows' loads are issued before the first row's math. MINB =
// the launch-bounds residency target (registers per thread <= 64K / (256 MINB)).
template <int VPL, int NR, int MINB>
__global__ void __launch_bounds__(256, MINB) k_ln_quantize_rows(const __nv_bfloat16* __restrict__ x, int64_t rows,
                                                             int nvec, const float* __restrict__ gamma,
                                                             const float* __restrict__ beta, float eps,
                                                             __nv_bfloat16* __restrict__ h, int8_t* __restrict__ q,
                                                             float* __restrict__ state, float* __restrict__ mean_out,
                                                             float* __restrict__ rstd_out, uint32_t* err) {
  // gamma / beta staged once per block in shared memory (they are re-read for every row)
  __shared__ float4 gb_s[2 * 2 * 32 * VPL];
  for (int t = threadIdx.x; t < 2 * nvec; t += blockDim.x) {
    gb_s[t] = __ldg(reinterpret_cast<const float4*>(gamma) + t);
    gb_s[2 * 32 * VPL + t] = __ldg(reinterpret_cast<const float4*>(beta) + t);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const float inv_n = 1.0f / static_cast<float>(nvec * 8);
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += NR * warps) {
    uint4 v[NR][VPL];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int i = j * 32 + lane;
        const int64_t rr = row + r * warps;
        v[r][j] = (rr < rows && i < nvec) ? ld_stream(reinterpret_cast<const uint4*>(x) + rr * nvec + i)
                                          : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (row + r * warps < rows)
        ln_row<VPL>(v[r], row + r * warps, nvec, lane, inv_n, eps, gb_s, h, q, state, mean_out, rstd_out, err);
  }
}

template <int VPL, int NR, int MINB>
void launch_ln_rows_v(sb_handle h, const __nv_bfloat16* x, int64_t rows, int nvec, const float* gamma,
                      const float* beta, float eps, __nv_bfloat16* out, int8_t* q, float* state, float* mean,
                      float* rstd) {
  static int blocks_per_sm[16] = {};
  int& bps = blocks_per_sm[h->device & 15];
  if (bps == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_ln_quantize_rows<VPL, NR, MINB>, 256, 0) != cudaSuccess ||
        bps < 1)
      bps = 1;
  }
  const int64_t need = (rows + 8 * NR - 1) / (8 * NR);
  const int64_t blocks = std::min<int64_t>(need, static_cast<int64_t>(h->num_sms) * bps);
  h->launches++;
  k_ln_quantize_rows<VPL, NR, MINB><<<static_cast<unsigned>(blocks), 256, 0, h->stream>>>(
      x, rows, nvec, gamma, beta, eps, out, q, state, mean, rstd, h->d_err);
}

// 2 rows per warp step at 2 blocks / SM measured best at 65792 x 1280 (89-90 us, 72% of HBM);
// 3 rows at 2 blocks: 91 us; 2 rows at 3 blocks (80 registers, spills): 94 us; 1 row at 3 or 4
// blocks: 115-117 us; 3-4 rows at 1 block: 122-125 us.
template <int VPL>
void launch_ln_rows(sb_handle h, const __nv_bfloat16* x, int64_t rows, int nvec, const float* gamma, const float* beta,
                    float eps, __nv_bfloat16* out, int8_t* q, float* state, float* mean, float* rstd) {
  launch_ln_rows_v<VPL, 2, 2>(h, x, rows, nvec, gamma, beta, eps, out, q, state, mean, rstd);
}

// LayerNorm backward for the fused pre-norm path (bf16 dh, x; fp32 mean, rstd, gamma):
//   xhat = (x - mean) rstd, g = dh gamma, dx = rstd (g - mean(g) - xhat mean(g xhat)),
//   dgamma = sum_rows dh xhat, dbeta = sum_rows dh.
// One warp per row (rows of <= 1280 columns, held in registers with their per-column gamma /
// beta-gradient accumulators); warp w owns rows w, w + W, ... and writes its column partials
// to part[w][...]; k_ln_bwd_reduce sums them over w in a fixed order (deterministic).
template <int VPL>
__device__ __forceinline__ void ln_bwd_row(const uint4 (&vx)[VPL], const uint4 (&vd)[VPL], int64_t row, int nvec,
                                           int lane, float inv_n, const float* __restrict__ mean,
                                           const float* __restrict__ rstd, const float2* gs, float2* accg,
                                           float2* accb, __nv_bfloat16* __restrict__ dx) {
  const int64_t off = row * static_cast<int64_t>(nvec);
  const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
  const float2 nmu = make_float2(-mu, -mu), rs2 = make_float2(rs, rs);
  float2 s1 = make_float2(0.0f, 0.0f), s2 = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int i = j * 32 + lane;
    if (i >= nvec) continue;
    const __nv_bfloat162* px = reinterpret_cast<const __nv_bfloat162*>(&vx[j]);
    const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&vd[j]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 fd = __bfloat1622float2(pd[k]);
      const float2 xh = __fmul2_rn(__fadd2_rn(__bfloat1622float2(px[k]), nmu), rs2);
      const float2 g = __fmul2_rn(fd, gs[k * nvec + i]);
      s1 = __fadd2_rn(s1, g);
      s2 = __ffma2_rn(g, xh, s2);
      accg[k * nvec + i] = __ffma2_rn(fd, xh, accg[k * nvec + i]);
      accb[k * nvec + i] = __fadd2_rn(accb[k * nvec + i], fd);
    }
  }
  float t1 = s1.x + s1.y, t2 = s2.x + s2.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    t1 += __shfl_xor_sync(0xffffffffu, t1, o);
    t2 += __shfl_xor_sync(0xffffffffu, t2, o);
  }
  const float2 nm1 = make_float2(-t1 * inv_n, -t1 * inv_n), nm2 = make_float2(-t2 * inv_n, -t2 * inv_n);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int i = j * 32 + lane;
    if (i >= nvec) continue;
    const __nv_bfloat162* px = reinterpret_cast<const __nv_bfloat162*>(&vx[j]);
    const __nv_bfloat162* pd = reinterpret_cast<const __nv_bfloat162*>(&vd[j]);
    uint4 o;
    __nv_bfloat162* po = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 xh = __fmul2_rn(__fadd2_rn(__bfloat1622float2(px[k]), nmu), rs2);
      const float2 g = __fmul2_rn(__bfloat1622float2(pd[k]), gs[k * nvec + i]);
      // rs (g - mean(g) - xhat mean(g xhat))
      po[k] = __float22bfloat162_rn(__fmul2_rn(__ffma2_rn(xh, nm2, __fadd2_rn(g, nm1)), rs2));
    }
    reinterpret_cast<uint4*>(dx)[off + i] = o;
  }
}

template <int VPL, int NR>
__global__ void __launch_bounds__(256) k_ln_backward_rows(const __nv_bfloat16* __restrict__ dh,
                                                          const __nv_bfloat16* __restrict__ x, int64_t rows, int nvec,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ rstd,
                                                          const float* __restrict__ gamma,
                                                          __nv_bfloat16* __restrict__ dx, float* __restrict__ part) {
  // shared: gamma as float2 [4][nvec] (column pair kk of vector i at kk * nvec + i: lane-consecutive,
  // conflict-free 8-byte accesses), then per warp its column accumulators dgamma, dbeta in the same
  // layout. The element math runs on the packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2).
  extern __shared__ float lnb_s[];
  float2* gs = reinterpret_cast<float2*>(lnb_s);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float2* accg = reinterpret_cast<float2*>(lnb_s + 8 * nvec * (1 + 2 * wib));
  float2* accb = accg + 4 * nvec;
  for (int t = threadIdx.x; t < 8 * nvec; t += blockDim.x)  // column t = 8 i + k
    lnb_s[2 * (((t & 7) >> 1) * nvec + (t >> 3)) + (t & 1)] = __ldg(gamma + t);
  for (int t = lane; t < 4 * nvec; t += 32) {
    accg[t] = make_float2(0.0f, 0.0f);
    accb[t] = make_float2(0.0f, 0.0f);
  }
  __syncthreads();
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int cols = nvec * 8;
  const float inv_n = 1.0f / static_cast<float>(cols);
  for (int64_t row = gw; row < rows; row += NR * warps) {
    uint4 vx[NR][VPL], vd[NR][VPL];
#pragma unroll
    for (int r = 0; r < NR; ++r)
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int i = j * 32 + lane;
        const int64_t rr = row + r * warps;
        const bool ok = rr < rows && i < nvec;
        vx[r][j] = ok ? ld_stream(reinterpret_cast<const uint4*>(x) + rr * nvec + i) : make_uint4(0, 0, 0, 0);
        vd[r][j] = ok ? ld_stream(reinterpret_cast<const uint4*>(dh) + rr * nvec + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
    for (int r = 0; r < NR; ++r)
      if (row + r * warps < rows)
        ln_bwd_row<VPL>(vx[r], vd[r], row + r * warps, nvec, lane, inv_n, mean, rstd, gs, accg, accb, dx);
  }
  // the block sums its warps' column accumulators in warp order (deterministic) and writes one
  // partial per block, in column order c = i * 8 + k
  __syncthreads();
  const int nw = blockDim.x >> 5;
  float* pg = part + static_cast<int64_t>(blockIdx.x) * 2 * cols;
  for (int t = threadIdx.x; t < 16 * nvec; t += blockDim.x) {
    const int which = t / (8 * nvec), tt = t - which * 8 * nvec;  // 0: dgamma, 1: dbeta
    float acc = 0.0f;
    for (int w = 0; w < nw; ++w) acc += lnb_s[8 * nvec * (1 + 2 * w + which) + tt];
    // float tt = 2 (kk nvec + i) + e holds column 8 i + 2 kk + e
    const int kk = tt / (2 * nvec), rem = tt - kk * 2 * nvec;
    pg[which * cols + (rem >> 1) * 8 + 2 * kk + (rem & 1)] = acc;
  }
}

template <int VPL, int NR>
void launch_ln_bwd_v(sb_handle h, int64_t blocks, size_t smem, const __nv_bfloat16* D, const __nv_bfloat16* X,
                     int64_t rows, int nvec, const float* mean, const float* rstd, const float* gamma, __nv_bfloat16* O,
                     float* part) {
  static bool attr[16] = {};  // one flag per instantiation and device
  if (!attr[h->device & 15]) {
    cudaFuncSetAttribute(k_ln_backward_rows<VPL, NR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr[h->device & 15] = true;
  }
  k_ln_backward_rows<VPL, NR><<<static_cast<unsigned>(blocks), 256, smem, h->stream>>>(D, X, rows, nvec, mean, rstd,
                                                                                       gamma, O, part);
}

// one row per warp step, 8-warp blocks, 2 per SM: loading two rows ahead measured slower (121.7
// vs 113.5 us at 65792 x 1280; 128 registers), and so did smaller blocks with more of them per
// SM (4 warps x 4 blocks: 119.7 us; 3 warps x 6 blocks: 139 us)
template <int VPL>
void launch_ln_bwd(sb_handle h, int64_t blocks, size_t smem, const __nv_bfloat16* D, const __nv_bfloat16* X,
                   int64_t rows, int nvec, const float* mean, const float* rstd, const float* gamma, __nv_bfloat16* O,
                   float* part) {
  launch_ln_bwd_v<VPL, 1>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part);
}

// Column sums of the per-block partials [nparts][2 * cols]: block = 32 columns x 8 warps; warp w
// sums partials w, w + 8, ... (coalesced 128-byte rows), then lane-wise over the 8 warps in
// order: deterministic.
__global__ void __launch_bounds__(256) k_ln_bwd_reduce(const float* __restrict__ part, int64_t nparts, int cols,
                                                       float* __restrict__ dgamma, float* __restrict__ dbeta) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.0f;
  if (c < 2 * cols)
    for (int64_t p = w; p < nparts; p += 8) s += part[p * 2 * cols + c];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < 2 * cols) {
    float t = 0.0f;
    for (int i = 0; i < 8; ++i) t += red[i][lane];
    if (c < cols) {
      if (dgamma) dgamma[c] = t;
    } else if (dbeta) {
      dbeta[c - cols] = t;
    }
  }
}

// SB_QUANT_KERNEL=tma selects the smem-ring kernel (A/B measurements); default: registers.
bool prefer_tma_ring() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SB_QUANT_KERNEL");
    v = (e && e[0] == 't') ? 1 : 0;
  }
  return v == 1;
}

template <typename T>
cudaError_t rowwise_impl(sb_handle h, const T* x, int64_t rows, int64_t cols, int64_t ldx, int8_t* q, int64_t ldq,
                         float* state) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int OUTB = VEC;  // bytes of payload per vector
  const bool vec_ok = (cols % VEC == 0) && (ldx % VEC == 0) && sb::aligned(x, 16) && (ldq % OUTB == 0) &&
                      sb::aligned(q, OUTB);
  h->launches++;
  if (!vec_ok) {
    const dim3 grid(static_cast<unsigned>((rows + 7) / 8));
    k_quantize_rowwise_scalar<T><<<grid, 256, 0, h->stream>>>(x, rows, cols, ldx, q, ldq, state, h->d_err);
    return cudaGetLastError();
  }
  if (!prefer_tma_ring() && cols / VEC <= 32 * 24 && rows > 0 &&
      rowwise_reg<T>(h, x, rows, static_cast<int>(cols / VEC), ldx, q, ldq, state))
    return cudaGetLastError();
  const int64_t row_bytes = cols * static_cast<int64_t>(sizeof(T));
  const int slot = static_cast<int>((row_bytes + 127) / 128 * 128);
  int stages = static_cast<int>(std::min<int64_t>(32, kQRingBytes / std::max(slot, 1)));
  if (stages > kQWarps) stages -= stages % kQWarps;  // slot ownership: see k_quantize_rowwise_tma
  if (stages >= 4) {
    static bool attr[16] = {};  // per device context
    const int smem = stages * slot + 2 * stages * 8;
    if (!attr[h->device & 15]) {
      cudaFuncSetAttribute(k_quantize_rowwise_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, kQRingBytes + 1024);
      attr[h->device & 15] = true;
    }
    int64_t blocks = std::min<int64_t>(rows, static_cast<int64_t>(h->num_sms) * 2);
    k_quantize_rowwise_tma<T><<<static_cast<unsigned>(blocks), kQThreads, smem, h->stream>>>(
        x, rows, cols, ldx, q, ldq, state, h->d_err, stages, slot);
  } else {
    const dim3 grid(static_cast<unsigned>((rows + 7) / 8));
    k_quantize_rowwise_stream<T><<<grid, 256, 0, h->stream>>>(x, rows, cols, ldx, q, ldq, state, h->d_err);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2 ----
// Tensor absmax: grid-stride over rows (warp per row), block max, one atomicMax per block.
template <typename T>
__global__ void __launch_bounds__(256) k_absmax_tensor(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ldx, unsigned int* word) {
  __shared__ uint32_t wmax[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t m = 0;
  const bool vec = (cols % (16 / sizeof(T)) == 0) && (ldx % (16 / sizeof(T)) == 0) && sb::aligned(x, 16);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + warp; r < rows; r += static_cast<int64_t>(gridDim.x) * 8) {
    const T* xr = x + r * ldx;
    if (vec) {
      const uint4* xv = reinterpret_cast<const uint4*>(xr);
      const int64_t nvec = cols / (16 / sizeof(T));
      for (int64_t v = lane; v < nvec; v += 32) m = max(m, vec_absmax_bits<T>(__ldg(xv + v)));
    } else {
      for (int64_t j = lane; j < cols; j += 32) m = max(m, abs_bits<T>(xr[j]));
    }
  }
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) wmax[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t b = 0;
    for (int i = 0; i < 8; ++i) b = max(b, wmax[i]);
    atomicMax(word, b);
  }
}

// Row absmax only (fp8 row axis): one warp per row.
template <typename T>
__global__ void __launch_bounds__(256) k_absmax_rows(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                                      unsigned int* words) {
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const T* xr = x + row * ldx;
  uint32_t m = 0;
  for (int64_t j = lane; j < cols; j += 32) m = max(m, abs_bits<T>(xr[j]));
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) words[row] = m;
}

// ------------------------------------------------------------------ K4 ----
// Column absmax: block = 32 columns x 8 row-lanes; grid.y splits rows; atomicMax per column.
template <typename T>
__global__ void __launch_bounds__(256) k_absmax_columns(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                         int64_t ldx, unsigned int* words) {
  __shared__ uint32_t part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + tx;
  uint32_t m = 0;
  if (col < cols)
    for (int64_t r = static_cast<int64_t>(blockIdx.y) * 8 + ty; r < rows; r += static_cast<int64_t>(gridDim.y) * 8)
      m = max(m, abs_bits<T>(x[r * ldx + col]));
  part[ty][tx] = m;
  __syncthreads();
  if (ty == 0 && col < cols) {
    for (int i = 1; i < 8; ++i) m = max(m, part[i][tx]);
    atomicMax(words + col, m);
  }
}

// ------------------------------------------------------------------ K3 ----
// Quantize with tensor (one word) or per-column states. 64x64 tile per block: the
// row-major payload is written straight out, the transposed payload goes through a
// shared-memory tile so both layouts come from a single read of x (quantize.cpp:154-157).
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_from_words(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                              int64_t ldx, const unsigned int* __restrict__ words,
                                                              int per_column, int8_t* __restrict__ q, int64_t ldq,
                                                              int8_t* __restrict__ qt, int64_t ldqt,
                                                              float* __restrict__ state, uint32_t* err) {
  __shared__ int8_t tile[64][64 + 4];
  const int tx = threadIdx.x & 15;  // 4 columns each
  const int ty = threadIdx.x >> 4;  // 16 rows per pass
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 64, c0 = static_cast<int64_t>(blockIdx.x) * 64;
  // tensor state (or this thread's 4 column states)
  uint32_t wb[4];
  float st[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t c = c0 + tx * 4 + i;
    wb[i] = per_column ? (c < cols ? words[c] : 0u) : words[0];
    st[i] = state_from_bits(wb[i]);
  }
  const bool bad = (wb[0] >= kNonFiniteBits) || (wb[1] >= kNonFiniteBits) || (wb[2] >= kNonFiniteBits) ||
                   (wb[3] >= kNonFiniteBits);
  if (bad) raise_nonfinite(err);
  // publish states once
  if (blockIdx.y == 0) {
    if (per_column) {
      if (ty == 0)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t c = c0 + tx * 4 + i;
          if (c < cols) state[c] = wb[i] >= kNonFiniteBits ? __uint_as_float(wb[i]) : st[i];
        }
    } else if (blockIdx.x == 0 && threadIdx.x == 0) {
      state[0] = wb[0] >= kNonFiniteBits ? __uint_as_float(wb[0]) : st[0];
    }
  }
  Scale sc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) sc[i] = make_scale(st[i]);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int lr = p * 16 + ty;
    const int64_t r = r0 + lr;
    uint32_t packed = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t c = c0 + tx * 4 + i;
      int8_t v = 0;
      if (r < rows && c < cols) v = quantize_one(x[r * ldx + c], sc[i]);
      tile[lr][tx * 4 + i] = v;
      packed |= static_cast<uint32_t>(static_cast<uint8_t>(v)) << (8 * i);
    }
    if (q && r < rows) {
      const int64_t c = c0 + tx * 4;
      if (c + 3 < cols && ((ldq & 3) == 0) && sb::aligned(q, 4)) {
        *reinterpret_cast<uint32_t*>(q + r * ldq + c) = packed;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (c + i < cols) q[r * ldq + c + i] = tile[lr][tx * 4 + i];
      }
    }
  }
  if (!qt) return;
  __syncthreads();
  // transposed: qt[c][r] = tile[r][c]; thread handles 4 consecutive r of one c
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int lc = p * 16 + ty;
    const int64_t c = c0 + lc;
    if (c >= cols) continue;
    const int64_t r = r0 + tx * 4;
    if (r + 3 < rows && ((ldqt & 3) == 0) && sb::aligned(qt, 4)) {
      uint32_t packed = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) packed |= static_cast<uint32_t>(static_cast<uint8_t>(tile[tx * 4 + i][lc])) << (8 * i);
      *reinterpret_cast<uint32_t*>(qt + c * ldqt + r) = packed;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (r + i < rows) qt[c * ldqt + r + i] = tile[tx * 4 + i][lc];
    }
  }
}

// ------------------------------------------------------------- K2+K3 fused ----
// Tensor-wise quantize (+ transposed payload) in ONE launch, as an ordered task list fetched
// from an atomic counter: first the absmax tasks (64-row slabs, atomicMax of bit patterns
// into sync[0], completion counted in sync[2]), then the 64 x 64 quantize tiles, which wait
// for the count and re-read x from L2 (W is <= tens of MB), writing q and/or q_t from one read
// (quantize.cpp:139-159). A tile task only ever waits on absmax tasks fetched before it by
// running blocks, so no co-residency is assumed (safe next to other kernels on other streams).
// bf16 input takes the one-FMA exact path (qvec_bf16_fast: the tensor state is a bf16 value
// >= every |x|). sync[0..3] are zeroed by the launcher (sync[1] task counter, sync[3] "state
// written" flag).
__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) k_quantize_tensorwise_fused(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                                    int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                    int8_t* __restrict__ qt, int64_t ldqt,
                                                                    float* __restrict__ state, unsigned int* sync,
                                                                    uint32_t* err) {
  constexpr int VEC = 16 / sizeof(T);
  __shared__ uint32_t red[8];
  __shared__ int64_t s_task;
  __shared__ __align__(16) int8_t tile[64][64 + 16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int vpr = static_cast<int>(cols / VEC);  // vectors per row
  // phase-1 tasks: absmax over slabs of ~32 KB of whole rows
  const int64_t slab_ = 32768 / (cols * static_cast<int64_t>(sizeof(T)));
  const int slab = static_cast<int>(slab_ > 1 ? slab_ : 1);
  const int64_t n_abs = (rows + slab - 1) / slab;
  const int64_t tr = (rows + 63) / 64, tc = (cols + 63) / 64;
  const int64_t n_tasks = n_abs + tr * tc;
  bool have_state = false;
  float st = 0.0f;
  Scale sc{};
  bool fast = false;
  sbptx::pdl_trigger();
  sbptx::pdl_wait();
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(sync + 1, 1u);
    __syncthreads();
    const int64_t task = s_task;
    __syncthreads();
    if (task >= n_tasks) break;
    if (task < n_abs) {
      // ---- phase 1 task: absmax of rows [slab task, slab task + slab)
      const int64_t r0 = task * slab;
      const int nr = static_cast<int>(rows - r0 < slab ? rows - r0 : slab);
      uint32_t m = 0;
      const int cnt = nr * vpr;
      // all of a step's loads in flight before the first use (ld_stream is volatile asm, so a
      // load-then-max loop would serialise one L2/HBM round trip per vector)
      for (int base = 0; base < cnt; base += 8 * 256) {
        uint4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int i = base + j * 256 + static_cast<int>(threadIdx.x);
          const int r = i / vpr, c = i - r * vpr;
          v[j] = i < cnt ? ld_stream(reinterpret_cast<const uint4*>(x + (r0 + r) * ldx) + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) m = max(m, vec_absmax_bits<T>(v[j]));
      }
      m = __reduce_max_sync(0xffffffffu, m);
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 1; i < 8; ++i) m = max(m, red[i]);
        if (m) atomicMax(sync, m);
        __threadfence();
        atomicAdd(sync + 2, 1u);
      }
      __syncthreads();
      continue;
    }
    // ---- phase 2 task: one 64 x 64 tile; every phase-1 task was fetched before this one by
    // a running block, so the wait below always ends (no co-residency assumption)
    if (!have_state) {
      if (threadIdx.x == 0) {
        while (ld_acquire_gpu(sync + 2) < static_cast<uint32_t>(n_abs)) __nanosleep(64);
        red[0] = ld_acquire_gpu(sync);
      }
      __syncthreads();
      const uint32_t wb = red[0];
      __syncthreads();
      if (wb >= kNonFiniteBits) {
        if (threadIdx.x == 0 && atomicOr(sync + 3, 1u) == 0u) {
          raise_nonfinite(err);
          state[0] = __uint_as_float(wb);
        }
        break;
      }
      st = state_from_bits(wb);
      if (threadIdx.x == 0 && atomicOr(sync + 3, 1u) == 0u) state[0] = st;
      sc = make_scale(st);
      fast = sizeof(T) == 2 && sc.pre == 1.0f;
      have_state = true;
    }
    const int64_t t = task - n_abs;
    const int64_t r0 = (t / tc) * 64, c0 = (t % tc) * 64;
    // 64 rows x 64 cols: thread -> (row lr = pass*32 + tid/8, 8-column group tid%8) for bf16,
    // (row pass*16 + tid/16, 4-column group tid%16) for fp32
    constexpr int GPR = 64 / VEC;          // vector groups per tile row
    constexpr int RPP = 256 / GPR;         // rows per pass
    const int g = threadIdx.x % GPR, lr0 = threadIdx.x / GPR;
    constexpr int NP = 64 / RPP;
    uint4 vin[NP];
#pragma unroll
    for (int pass = 0; pass < NP; ++pass) {  // both passes' loads in flight first
      const int64_t r = r0 + pass * RPP + lr0, c = c0 + g * VEC;
      vin[pass] = (r < rows && c < cols) ? ld_stream(reinterpret_cast<const uint4*>(x + r * ldx + c))
                                         : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int pass = 0; pass < NP; ++pass) {
      const int lr = pass * RPP + lr0;
      const int64_t r = r0 + lr, c = c0 + g * VEC;
      uint32_t w0 = 0, w1 = 0;  // payload bytes of this vector (VEC <= 8)
      if (r < rows && c < cols) {
        const uint4 v = vin[pass];
        if constexpr (sizeof(T) == 2) {
          const uint2 o = fast ? qvec_bf16_fast(v, sc.inv2) : VecQ<T>::run(v, sc);
          w0 = o.x;
          w1 = o.y;
        } else {
          w0 = VecQ<T>::run(v, sc);
        }
        if (q) {
          if constexpr (VEC == 8)
            *reinterpret_cast<uint2*>(q + r * ldq + c) = make_uint2(w0, w1);
          else
            *reinterpret_cast<uint32_t*>(q + r * ldq + c) = w0;
        }
      }
      if constexpr (VEC == 8)
        *reinterpret_cast<uint2*>(&tile[lr][g * 8]) = make_uint2(w0, w1);
      else
        *reinterpret_cast<uint32_t*>(&tile[lr][g * 4]) = w0;
    }
    if (qt) {
      __syncthreads();
      // q_t[c][r0 .. r0+63]: thread -> column lc = tid / 4, 16 consecutive rows (tid % 4) * 16
      const int lc = threadIdx.x >> 2, rq = (threadIdx.x & 3) * 16;
      const int64_t c = c0 + lc;
      if (c < cols) {
        uint32_t wv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          uint32_t pk = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) pk |= static_cast<uint32_t>(static_cast<uint8_t>(tile[rq + 4 * k + i][lc])) << (8 * i);
          wv[k] = pk;
        }
        const int64_t r = r0 + rq;
        int8_t* dst = qt + c * ldqt + r;
        if (r + 15 < rows && sb::aligned(dst, 16)) {
          *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        } else {
          for (int i = 0; i < 16 && r + i < rows; ++i) dst[i] = static_cast<int8_t>((wv[i >> 2] >> (8 * (i & 3))) & 0xff);
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------- K2+K3 one pass ----
// Tensor-wise quantize (+ transposed payload) for weights that fit on the chip at once: one
// 128-row tile per block (bf16: 128 x 128, fp32: 128 x 64; 2048 16-byte vectors, 8 per thread)
// held in registers across a grid-wide absmax: each block loads its tile with all loads in
// flight, max-reduces it into sync[0] and counts itself done in sync[2]; once every block has
// arrived it quantizes the registers (one HBM read of W in total) and writes q row-major and
// q_t through a shared-memory transpose. The launch is cooperative (the runtime guarantees the
// blocks are co-resident, or refuses the launch and the task-list kernel above runs instead).
// ~2 HBM round trips + one grid barrier instead of the task list's serial atomics / barriers
// per 8 KB task (22 us -> a few us for the ViT-H weights).
constexpr int kTwRows = 128;
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_tensorwise_coop(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                                   int64_t ldx, int8_t* __restrict__ q, int64_t ldq,
                                                                   int8_t* __restrict__ qt, int64_t ldqt,
                                                                   float* __restrict__ state, unsigned int* sync,
                                                                   uint32_t* err) {
  constexpr int VEC = 16 / sizeof(T);
  constexpr int TC = 16 * VEC;  // tile columns: 16 vectors per tile row
  __shared__ uint32_t red[8];
  __shared__ __align__(16) int8_t tile[kTwRows][TC + 16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tc = (cols + TC - 1) / TC;
  const int64_t r0 = (blockIdx.x / tc) * kTwRows, c0 = (blockIdx.x % tc) * TC;
  const int vc = threadIdx.x & 15, lr0 = threadIdx.x >> 4;  // vector column, first tile row (+16 j)
  const int64_t c = c0 + vc * VEC;
  sbptx::pdl_trigger();
  sbptx::pdl_wait();
  uint4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t r = r0 + lr0 + 16 * j;
    v[j] = (r < rows && c < cols) ? ld_stream(reinterpret_cast<const uint4*>(x + r * ldx + c)) : make_uint4(0, 0, 0, 0);
  }
  uint32_t m = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) m = max(m, vec_absmax_bits<T>(v[j]));
  m = __reduce_max_sync(0xffffffffu, m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < 8; ++i) m = max(m, red[i]);
    if (m) atomicMax(sync, m);
    __threadfence();
    atomicAdd(sync + 2, 1u);
    while (ld_acquire_gpu(sync + 2) < gridDim.x) __nanosleep(32);
    red[0] = ld_acquire_gpu(sync);
  }
  __syncthreads();
  const uint32_t wb = red[0];
  if (wb >= kNonFiniteBits) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      raise_nonfinite(err);
      state[0] = __uint_as_float(wb);
    }
    return;
  }
  const float st = state_from_bits(wb);
  if (blockIdx.x == 0 && threadIdx.x == 0) state[0] = st;
  const Scale sc = make_scale(st);
  const bool fast = sizeof(T) == 2 && sc.pre == 1.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int lr = lr0 + 16 * j;
    const int64_t r = r0 + lr;
    uint32_t w0 = 0, w1 = 0;
    if constexpr (sizeof(T) == 2) {
      const uint2 o = fast ? qvec_bf16_fast(v[j], sc.inv2) : VecQ<T>::run(v[j], sc);
      w0 = o.x;
      w1 = o.y;
    } else {
      w0 = VecQ<T>::run(v[j], sc);
    }
    if (q && r < rows && c < cols) {
      if constexpr (VEC == 8)
        *reinterpret_cast<uint2*>(q + r * ldq + c) = make_uint2(w0, w1);
      else
        *reinterpret_cast<uint32_t*>(q + r * ldq + c) = w0;
    }
    if constexpr (VEC == 8)
      *reinterpret_cast<uint2*>(&tile[lr][vc * 8]) = make_uint2(w0, w1);
    else
      *reinterpret_cast<uint32_t*>(&tile[lr][vc * 4]) = w0;
  }
  if (!qt) return;
  __syncthreads();
  // q_t[c][r0 .. r0 + 127]: 256 / TC threads per tile column, 16 rows (one uint4) per step
  constexpr int TPC = 256 / TC;            // threads per tile column (2 bf16, 4 fp32)
  constexpr int RPT = kTwRows / TPC;       // rows per thread (64 / 32)
  const int lc = threadIdx.x / TPC, rq0 = (threadIdx.x % TPC) * RPT;
  const int64_t cc = c0 + lc;
  if (cc >= cols) return;
#pragma unroll
  for (int k0 = 0; k0 < RPT; k0 += 16) {
    uint32_t wv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t pk = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) pk |= static_cast<uint32_t>(static_cast<uint8_t>(tile[rq0 + k0 + 4 * k + i][lc])) << (8 * i);
      wv[k] = pk;
    }
    const int64_t r = r0 + rq0 + k0;
    int8_t* dst = qt + cc * ldqt + r;
    if (r + 15 < rows && sb::aligned(dst, 16)) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    } else {
      for (int i = 0; i < 16 && r + i < rows; ++i) dst[i] = static_cast<int8_t>((wv[i >> 2] >> (8 * (i & 3))) & 0xff);
    }
  }
}

template <typename T>
bool launch_tensorwise_coop(sb_handle h, const T* x, int64_t rows, int64_t cols, int64_t ldx, int8_t* q, int64_t ldq,
                            int8_t* qt, int64_t ldqt, float* state, unsigned int* sync, cudaError_t* err) {
  constexpr int TC = 16 * (16 / sizeof(T));
  static int cap[16] = {};  // co-resident blocks per device
  const int d = h->device & 15;
  if (cap[d] == 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_quantize_tensorwise_coop<T>, 256, 0) != cudaSuccess || b < 1)
      b = 0;
    cudaGetLastError();
    cap[d] = b > 0 ? b * h->num_sms : -1;
  }
  const int64_t tiles = ((rows + kTwRows - 1) / kTwRows) * ((cols + TC - 1) / TC);
  if (cap[d] < 0 || tiles > cap[d]) return false;
  *err = cudaMemsetAsync(sync, 0, 4 * sizeof(unsigned int), h->stream);
  if (*err != cudaSuccess) return true;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(tiles));
  cfg.blockDim = dim3(256);
  cfg.stream = h->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  h->launches++;
  *err = cudaLaunchKernelEx(&cfg, k_quantize_tensorwise_coop<T>, x, rows, cols, ldx, q, ldq, qt, ldqt, state, sync,
                            h->d_err);
  if (*err == cudaErrorCooperativeLaunchTooLarge || *err == cudaErrorNotSupported) {
    cudaGetLastError();
    h->launches--;
    cap[d] = -1;  // never again on this device: the task-list kernel runs
    return false;
  }
  return true;
}

// ----------------------------------------------------------------- K10 ----
template <typename TO>
__device__ __forceinline__ TO from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

template <typename TO>
__global__ void k_dequantize(const int8_t* __restrict__ q, int64_t rows, int64_t cols, int64_t ldq,
                             const float* __restrict__ state, int axis, TO* __restrict__ y, int64_t ldy) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float s = axis == 0 ? state[r] : axis == 1 ? state[c] : state[0];
    // float(double(p) * double(s) / 127.0), quantize.cpp:191-194
    const double d = __ddiv_rn(__dmul_rn(static_cast<double>(q[r * ldq + c]), static_cast<double>(s)), 127.0);
    y[r * ldy + c] = from_f32<TO>(__double2float_rn(d));
  }
}

// ------------------------------------------------------------------ K8 ----
// fp8 snap with ties to the smaller magnitude and saturation at the set edges; returns
// the e4m3 (bias 7, max 448, S.1111.111 = NaN) / e5m2 (bias 15, max 57344) byte.
// Integer-only (no FRND / F2I, which run on the 16/clk/SM conversion pipe): with a = |r| =
// M 2^(E-150) (M the 24-bit significand, E the biased exponent), the normal-grid code drops
// 23-MB mantissa bits rounding half toward zero; below 2^(1-BIAS) the denormal grid step is
// 2^(1-BIAS-MB), so code = M / 2^(151-BIAS-MB-E) rounded half down (shift clamped to 31:
// everything under a quarter of the smallest step is 0). Checked against the float-path
// formulation on every non-negative f32 (tools/fp8_div_check.cu).
template <int MB, int BIAS>
__device__ __forceinline__ uint8_t fp8_snap_encode(float r, float maxv, uint32_t maxcode) {
  const uint32_t bits = __float_as_uint(r);
  const uint32_t sign = (bits >> 31) << 7;
  const uint32_t ab = bits & 0x7fffffffu;
  constexpr uint32_t drop = 23 - MB;
  const uint32_t code_n = ((ab + (1u << (drop - 1)) - 1u) >> drop) - ((127u - BIAS) << MB);
  const uint32_t E = ab >> 23;
  const uint32_t M = (ab & 0x7fffffu) | 0x800000u;
  const uint32_t sh = min(31u, static_cast<uint32_t>(151 - BIAS - MB) - min(E, static_cast<uint32_t>(151 - BIAS - MB - 1)));
  const uint32_t code_d = (M + (1u << (sh - 1)) - 1u) >> sh;
  uint32_t code = E < static_cast<uint32_t>(128 - BIAS) ? code_d : code_n;
  code = ab >= __float_as_uint(maxv) ? maxcode : code;
  return static_cast<uint8_t>(sign | code);
}

// The same code for |r| <= 1 (every quotient x / max|x|), no saturation branch, with the
// denormal grid done on the FMA pipe: n = |r| 2^(BIAS+MB-1) (exact), t = RNE(n) via the
// 1.5*2^23 magic, minus 1 where RNE rounded an exact .5 up (residual n - t == -1/2): that is
// round half down. Integer work: 2 ops for the normal grid, 1 for the denormal, 2 to select,
// 2 for the sign (vs ~17 integer ops in fp8_snap_encode). Checked against it on every f32
// with |r| <= 1 (tools/fp8_div_check.cu).
template <int MB, int BIAS>
__device__ __forceinline__ uint32_t fp8_snap_unit(float r) {
  const uint32_t bits = __float_as_uint(r);
  const uint32_t ab = bits & 0x7fffffffu;
  constexpr uint32_t drop = 23 - MB;
  const uint32_t code_n = ((ab + (1u << (drop - 1)) - 1u) >> drop) - ((127u - BIAS) << MB);
  const float n = __fmul_rn(__uint_as_float(ab), __uint_as_float(static_cast<uint32_t>(127 + BIAS + MB - 1) << 23));
  const float m = __fadd_rn(n, 12582912.0f);
  const float rn = __fsub_rn(m, 12582912.0f);
  const uint32_t code_d = (__float_as_uint(m) - 0x4B400000u) - (__fsub_rn(n, rn) == -0.5f ? 1u : 0u);
  const uint32_t code = ab < (static_cast<uint32_t>(128 - BIAS) << 23) ? code_d : code_n;
  return ((bits >> 24) & 0x80u) | code;
}

// fp8_snap_unit without the sign: a = |ratio| >= 0.
template <int MB, int BIAS>
__device__ __forceinline__ uint32_t fp8_code_unit_abs(float a) {
  const uint32_t ab = __float_as_uint(a);
  constexpr uint32_t drop = 23 - MB;
  const uint32_t code_n = ((ab + (1u << (drop - 1)) - 1u) >> drop) - ((127u - BIAS) << MB);
  const float n = __fmul_rn(a, __uint_as_float(static_cast<uint32_t>(127 + BIAS + MB - 1) << 23));
  const float m = __fadd_rn(n, 12582912.0f);
  const float rn = __fsub_rn(m, 12582912.0f);
  const uint32_t code_d = (__float_as_uint(m) - 0x4B400000u) - (__fsub_rn(n, rn) == -0.5f ? 1u : 0u);
  return ab < (static_cast<uint32_t>(128 - BIAS) << 23) ? code_d : code_n;
}

__device__ __forceinline__ float fp8_decode(uint8_t b, int fmt) {
  const uint32_t s = (b >> 7) & 1u;
  float v;
  if (fmt == 0) {  // e4m3
    const uint32_t e = (b >> 3) & 0xFu, m = b & 7u;
    v = e == 0 ? ldexpf(static_cast<float>(m), -9) : ldexpf(1.0f + m / 8.0f, static_cast<int>(e) - 7);
  } else {  // e5m2
    const uint32_t e = (b >> 2) & 0x1Fu, m = b & 3u;
    v = e == 0 ? ldexpf(static_cast<float>(m), -16) : ldexpf(1.0f + m / 4.0f, static_cast<int>(e) - 15);
  }
  return s ? -v : v;
}

template <typename T>
__global__ void k_quantize_fp8(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx, int fmt, int axis,
                               const unsigned int* __restrict__ words, uint8_t* __restrict__ q, int64_t ldq,
                               float* __restrict__ state, uint32_t* err) {
  const int64_t n = rows * cols;
  const int64_t nstate = axis == 0 ? rows : axis == 1 ? cols : 1;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = tid; i < nstate; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t w = words[i];
    if (w >= kNonFiniteBits) raise_nonfinite(err);
    state[i] = w >= kNonFiniteBits ? __uint_as_float(w) : state_from_bits(w);
  }
  for (int64_t i = tid; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const uint32_t w = words[axis == 0 ? r : axis == 1 ? c : 0];
    const float s = state_from_bits(w);
    // f32(double(x)/double(s)) == __fdiv_rn(x, s) (innocuous double rounding, 53 >= 2*24+2)
    const float ratio = __fdiv_rn(to_f32(x[r * ldx + c]), s);
    q[r * ldq + c] = fmt == 0 ? fp8_snap_encode<3, 7>(ratio, 448.0f, 0x7Eu)
                              : fp8_snap_encode<2, 15>(ratio, 57344.0f, 0x7Bu);
  }
}


// fp8 payload of one 16-byte input vector with a row / tensor state (8 bf16 -> 8 bytes, 4 f32 -> 4).
// ratio = f32(double(x)/double(s)) == __fdiv_rn(x, s) (innocuous double rounding, 53 >= 2*24+2).
//
// bf16 x with a state s in [2^-60, 2^64]: fl32(x/s) is formed as q0 = x * r, r = fl32(1/s),
// plus one Markstein correction q = fma(fma(-s, q0, x), r, q0) with the sign of x restored
// (so -0 stays -0). The fp8 payload this gives equals the one from the correctly rounded
// quotient for EVERY bf16 pair |x| <= s in that range, e4m3 and e5m2 (exhaustive check,
// tools/fp8_div_check.cu, ~1.07e9 pairs); rows outside it and fp32 input use __fdiv_rn.
// bf16 fast path on magnitudes: the quotient of |x| (abs is a free operand modifier), the
// magnitude code, and the 8 sign bits OR-ed in from the raw bf16 words at the end.
// fp8_code_unit_abs for two magnitudes at once, the float steps on the packed fp32x2 pipe
// (FFMA2 / FADD2: per lane the same IEEE operations, so the codes are identical):
//   normal:    ((|a| + half - 1) >> drop) - (127 - BIAS) << MB, folded into one add;
//   subnormal: round-half-down(n), n = |a| 2^(BIAS+MB-1) < 2^MB, as ceil(n - 1/2): n - 1/2 is
//              exact (one FFMA), ceil by the magic-number add rounded toward +inf.
template <int MB, int BIAS>
__device__ __forceinline__ void fp8_code2_abs(float2 a, uint32_t& c0, uint32_t& c1) {
  constexpr uint32_t drop = 23 - MB;
  constexpr uint32_t K = (1u << (drop - 1)) - 1u - (static_cast<uint32_t>(127 - BIAS) << 23);  // mod 2^32
  constexpr uint32_t thr = static_cast<uint32_t>(128 - BIAS) << 23;
  const float P = __uint_as_float(static_cast<uint32_t>(127 + BIAS + MB - 1) << 23);
  const float2 t = __ffma2_rn(a, make_float2(P, P), make_float2(-0.5f, -0.5f));
  const float2 m = __fadd2_ru(t, make_float2(12582912.0f, 12582912.0f));
  const uint32_t ab0 = __float_as_uint(a.x), ab1 = __float_as_uint(a.y);
  c0 = ab0 < thr ? __float_as_uint(m.x) - 0x4B400000u : (ab0 + K) >> drop;
  c1 = ab1 < thr ? __float_as_uint(m.y) - 0x4B400000u : (ab1 + K) >> drop;
}

// bf16 fast path on magnitudes, two elements per packed fp32x2 operation: |x| is the bf16 word
// with its sign bits cleared, the quotient |x| / s by q0 = |x| r and one Markstein correction,
// the magnitude codes packed with byte permutes and the 8 sign bits OR-ed in from the raw words.
template <int FMT>
__device__ __forceinline__ uint2 fp8_vec_bf16_fast(const uint4& v, float s, float r) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  const float2 r2 = make_float2(r, r), ns2 = make_float2(-s, -s);
  uint32_t c[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t wa = w[i] & 0x7fff7fffu;
    const float2 ax = make_float2(__uint_as_float(wa << 16), __uint_as_float(wa & 0xffff0000u));
    const float2 q0 = __fmul2_rn(ax, r2);
    const float2 a = __ffma2_rn(__ffma2_rn(ns2, q0, ax), r2, q0);
    if (FMT == 0)
      fp8_code2_abs<3, 7>(a, c[2 * i], c[2 * i + 1]);
    else
      fp8_code2_abs<2, 15>(a, c[2 * i], c[2 * i + 1]);
  }
  // sign of element 2k is bit 15 of w[k] (bit 7 of byte 1), of element 2k+1 bit 31 (byte 3)
  const uint32_t s0 = __byte_perm(w[0], w[1], 0x7531) & 0x80808080u;
  const uint32_t s1 = __byte_perm(w[2], w[3], 0x7531) & 0x80808080u;
  const uint32_t p0 = __byte_perm(__byte_perm(c[0], c[1], 0x0040), __byte_perm(c[2], c[3], 0x0040), 0x5410);
  const uint32_t p1 = __byte_perm(__byte_perm(c[4], c[5], 0x0040), __byte_perm(c[6], c[7], 0x0040), 0x5410);
  return make_uint2(p0 | s0, p1 | s1);
}

template <bool FAST, int FMT, typename T>
__device__ __forceinline__ uint2 fp8_vec(const uint4& v, float s, float r) {
  if constexpr (FAST && sizeof(T) == 2) return fp8_vec_bf16_fast<FMT>(v, s, r);
  constexpr int N = Unpack<T>::N;
  float x[N];
  Unpack<T>::run(v, x);
  uint32_t b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < N; ++i) {
    float ratio;
    if (FAST) {
      const float q0 = __fmul_rn(x[i], r);
      ratio = copysignf(__fmaf_rn(__fmaf_rn(-s, q0, x[i]), r, q0), x[i]);
    } else {
      ratio = __fdiv_rn(x[i], s);
    }
    if (FAST)  // |ratio| <= 1: the quotient's state is the slice absmax
      b[i] = FMT == 0 ? fp8_snap_unit<3, 7>(ratio) : fp8_snap_unit<2, 15>(ratio);
    else
      b[i] = FMT == 0 ? fp8_snap_encode<3, 7>(ratio, 448.0f, 0x7Eu) : fp8_snap_encode<2, 15>(ratio, 57344.0f, 0x7Bu);
  }
  return make_uint2(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24), b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24));
}
// bf16 with a state in [2^-60, 2^64] takes the FAST quotient (see above); anything else the
// correctly rounded division. `r` = fl32(1/s) or 0 for "exact division".
template <typename T>
__device__ __forceinline__ uint2 fp8_vec_any(const uint4& v, float s, int fmt, float r) {
  if (sizeof(T) == 2 && r != 0.0f) return fmt == 0 ? fp8_vec<true, 0, T>(v, s, r) : fp8_vec<true, 1, T>(v, s, r);
  return fmt == 0 ? fp8_vec<false, 0, T>(v, s, r) : fp8_vec<false, 1, T>(v, s, r);
}

// Row-axis fp8 quantize, one warp per row held in registers: absmax + state + payload in one
// pass over x (the register-resident design of k_quantize_rowwise_reg).
template <typename T, int VPL, int FMT>
__global__ void __launch_bounds__(256) k_quantize_fp8_rows_reg(const T* __restrict__ x, int64_t rows, int nvec,
                                                               int64_t ldx, int fmt, uint8_t* __restrict__ q,
                                                               int64_t ldq, float* __restrict__ state, uint32_t* err) {
  constexpr int OUTB = 16 / sizeof(T);  // payload bytes per vector
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * ldx);
    uint4 v[VPL];
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = j * 32 + lane;
      v[j] = i < nvec ? ld_stream(xr + i) : make_uint4(0, 0, 0, 0);
    }
    uint32_t amax = 0;
#pragma unroll
    for (int j = 0; j < VPL; ++j) amax = max(amax, vec_absmax_bits<T>(v[j]));
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        state[row] = __uint_as_float(amax);
      }
      continue;
    }
    const float st = state_from_bits(amax);
    if (lane == 0) state[row] = st;
    const float rcp = (st >= 0x1p-60f && st <= 0x1p64f) ? __frcp_rn(st) : 0.0f;  // 0: exact division
    uint8_t* qr = q + row * ldq;
    auto emit = [&](auto fast) {
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int i = j * 32 + lane;
        if (i < nvec) {
          const uint2 o = fp8_vec<decltype(fast)::value, FMT, T>(v[j], st, rcp);
          if (OUTB == 8)
            *reinterpret_cast<uint2*>(qr + i * 8) = o;
          else
            *reinterpret_cast<uint32_t*>(qr + i * 4) = o.x;
        }
      }
    };
    if (sizeof(T) == 2 && rcp != 0.0f)
      emit(std::true_type{});
    else
      emit(std::false_type{});
  }
}

// Tensor / column-axis fp8 quantize from absmax words, 16-byte vectors, rows grid-strided by
// block, no per-element integer division.
template <typename T>
__global__ void __launch_bounds__(256) k_quantize_fp8_vec(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                          int64_t ldx, int fmt, int axis,
                                                          const unsigned int* __restrict__ words,
                                                          uint8_t* __restrict__ q, int64_t ldq,
                                                          float* __restrict__ state, uint32_t* err) {
  constexpr int VEC = 16 / sizeof(T);
  const int64_t nstate = axis == 1 ? cols : 1;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nstate;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t w = words[i];
    if (w >= kNonFiniteBits) raise_nonfinite(err);
    state[i] = w >= kNonFiniteBits ? __uint_as_float(w) : state_from_bits(w);
  }
  const int64_t nv = cols / VEC;
  const float st = axis == 1 ? 0.0f : state_from_bits(words[0]);
  const float rcp = (axis != 1 && st >= 0x1p-60f && st <= 0x1p64f) ? __frcp_rn(st) : 0.0f;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + r * ldx);
    for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) {
      const uint4 xv = ld_stream(xr + v);
      uint2 o;
      if (axis == 1) {  // per-column states: VEC distinct divisors
        constexpr int N = Unpack<T>::N;
        float xs[N];
        Unpack<T>::run(xv, xs);
        uint32_t b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const float ratio = __fdiv_rn(xs[k], state_from_bits(__ldg(words + v * VEC + k)));
          b[k] = fmt == 0 ? fp8_snap_encode<3, 7>(ratio, 448.0f, 0x7Eu) : fp8_snap_encode<2, 15>(ratio, 57344.0f, 0x7Bu);
        }
        o = make_uint2(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24), b[4] | (b[5] << 8) | (b[6] << 16) | (b[7] << 24));
      } else {
        o = fp8_vec_any<T>(xv, st, fmt, rcp);
      }
      if (VEC == 8)
        *reinterpret_cast<uint2*>(q + r * ldq + v * 8) = o;
      else
        *reinterpret_cast<uint32_t*>(q + r * ldq + v * 4) = o.x;
    }
  }
}

// Long rows: two passes over the row per warp — absmax streaming (nothing kept), then reload
// (an L2 hit: the row was just read) and quantize. ~40 registers instead of 4 per 16-byte
// vector of the row, so 4x the resident warps hide the ALU-heavy snap's latency.
template <typename T, int FMT>
__global__ void __launch_bounds__(256) k_quantize_fp8_rows_2pass(const T* __restrict__ x, int64_t rows, int nvec,
                                                                 int64_t ldx, uint8_t* __restrict__ q, int64_t ldq,
                                                                 float* __restrict__ state, uint32_t* err) {
  constexpr int OUTB = 16 / sizeof(T);
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); row < rows;
       row += warps) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * ldx);
    uint32_t amax = 0;
#pragma unroll 4
    for (int i = lane; i < nvec; i += 32) amax = max(amax, vec_absmax_bits<T>(__ldcg(xr + i)));
    amax = __reduce_max_sync(0xffffffffu, amax);
    if (amax >= kNonFiniteBits) {
      if (lane == 0) {
        raise_nonfinite(err);
        state[row] = __uint_as_float(amax);
      }
      continue;
    }
    const float st = state_from_bits(amax);
    if (lane == 0) state[row] = st;
    const float rcp = (st >= 0x1p-60f && st <= 0x1p64f) ? __frcp_rn(st) : 0.0f;
    uint8_t* qr = q + row * ldq;
    auto emit = [&](auto fast) {
#pragma unroll 4
      for (int i = lane; i < nvec; i += 32) {
        const uint2 o = fp8_vec<decltype(fast)::value, FMT, T>(ld_stream(xr + i), st, rcp);
        if (OUTB == 8)
          *reinterpret_cast<uint2*>(qr + i * 8) = o;
        else
          *reinterpret_cast<uint32_t*>(qr + i * 4) = o.x;
      }
    };
    if (sizeof(T) == 2 && rcp != 0.0f)
      emit(std::true_type{});
    else
      emit(std::false_type{});
  }
}

template <typename T, int FMT>
bool fp8_rows_reg_f(sb_handle h, const T* x, int64_t rows, int nvec, int64_t ldx, int fmt, uint8_t* q, int64_t ldq,
                    float* state) {
  const int vpl = (nvec + 31) / 32;
  auto go = [&](auto kern) {
    static int bps = 0;
    if (bps == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0) != cudaSuccess || bps < 1))
      bps = 1;
    const int64_t blocks = std::min<int64_t>((rows + 7) / 8, static_cast<int64_t>(h->num_sms) * bps);
    kern<<<static_cast<unsigned>(blocks), 256, 0, h->stream>>>(x, rows, nvec, ldx, fmt, q, ldq, state, h->d_err);
    return true;
  };
  static int keep = -1;
  if (keep < 0) keep = getenv("SB_FP8_KEEP") ? atoi(getenv("SB_FP8_KEEP")) : 0;
  if (vpl > 6 && !keep) {
    auto kern = k_quantize_fp8_rows_2pass<T, FMT>;
    static int bps = 0;
    if (bps == 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, 256, 0) != cudaSuccess || bps < 1))
      bps = 1;
    const int64_t blocks = std::min<int64_t>((rows + 7) / 8, static_cast<int64_t>(h->num_sms) * bps);
    kern<<<static_cast<unsigned>(blocks), 256, 0, h->stream>>>(x, rows, nvec, ldx, q, ldq, state, h->d_err);
    return true;
  }
  switch (vpl) {
    case 1: return go(k_quantize_fp8_rows_reg<T, 1, FMT>);
    case 2: return go(k_quantize_fp8_rows_reg<T, 2, FMT>);
    case 3:
    case 4: return go(k_quantize_fp8_rows_reg<T, 4, FMT>);
    case 5:
    case 6: return go(k_quantize_fp8_rows_reg<T, 6, FMT>);
    case 7:
    case 8: return go(k_quantize_fp8_rows_reg<T, 8, FMT>);
    case 9:
    case 10:
    case 11:
    case 12: return go(k_quantize_fp8_rows_reg<T, 12, FMT>);
    case 13:
    case 14:
    case 15:
    case 16: return go(k_quantize_fp8_rows_reg<T, 16, FMT>);
    case 17:
    case 18:
    case 19:
    case 20: return go(k_quantize_fp8_rows_reg<T, 20, FMT>);
    default: return false;
  }
}
template <typename T>
bool fp8_rows_reg(sb_handle h, const T* x, int64_t rows, int nvec, int64_t ldx, int fmt, uint8_t* q, int64_t ldq,
                  float* state) {
  return fmt == 0 ? fp8_rows_reg_f<T, 0>(h, x, rows, nvec, ldx, fmt, q, ldq, state)
                  : fp8_rows_reg_f<T, 1>(h, x, rows, nvec, ldx, fmt, q, ldq, state);
}

template <typename TO>
__global__ void k_dequantize_fp8(const uint8_t* __restrict__ q, int64_t rows, int64_t cols, int64_t ldq, int fmt,
                                 const float* __restrict__ state, int axis, TO* __restrict__ y, int64_t ldy) {
  const int64_t n = rows * cols;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    const float s = axis == 0 ? state[r] : axis == 1 ? state[c] : state[0];
    // float(double(v) * double(s)) == __fmul_rn(v, s): the double product is exact
    y[r * ldy + c] = from_f32<TO>(__fmul_rn(fp8_decode(q[r * ldq + c], fmt), s));
  }
}

// fp8_cast (quantize.cpp:78-84): snap to the value set without a scale; non-finite -> latch.
__global__ void k_fp8_cast(const float* __restrict__ x, int64_t n, int fmt, float* __restrict__ y, uint32_t* err) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = x[i];
    if (!isfinite(v)) raise_nonfinite(err);
    const uint8_t b = fmt == 0 ? fp8_snap_encode<3, 7>(v, 448.0f, 0x7Eu) : fp8_snap_encode<2, 15>(v, 57344.0f, 0x7Bu);
    y[i] = fp8_decode(b, fmt);
  }
}

template <typename TI, typename TO>
__global__ void k_convert(const TI* __restrict__ x, TO* __restrict__ y, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = from_f32<TO>(to_f32(x[i]));
}

unsigned grid_for(int64_t n, int per_block, int num_sms) {
  int64_t g = (n + per_block - 1) / per_block;
  const int64_t cap = static_cast<int64_t>(num_sms) * 32;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace

namespace sb {

cudaError_t launch_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                    int8_t* q, int64_t ldq, float* state) {
  if (dt == SB_BF16)
    return rowwise_impl(h, static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, q, ldq, state);
  return rowwise_impl(h, static_cast<const float*>(x), rows, cols, ldx, q, ldq, state);
}

cudaError_t launch_absmax_tensor(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 unsigned int* word) {
  cudaError_t e = cudaMemsetAsync(word, 0, sizeof(unsigned int), h->stream);
  if (e != cudaSuccess) return e;
  const unsigned grid = grid_for(rows, 8, h->num_sms);
  h->launches++;
  if (dt == SB_BF16)
    k_absmax_tensor<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, word);
  else
    k_absmax_tensor<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, word);
  return cudaGetLastError();
}

// One-launch tensor-wise quantize when x is 16-byte vectorisable; false = use K2 + K3.
bool launch_quantize_tensorwise_fused(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                      int64_t ldx, int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state,
                                      unsigned int* sync, cudaError_t* err) {
  const int vec = dt == SB_BF16 ? 8 : 4;
  if (cols % vec || ldx % vec || !sb::aligned(x, 16) || rows <= 0 || cols <= 0) return false;
  if (q && (ldq % vec || !sb::aligned(q, 8))) return false;
  if (!getenv("SB_TW_TASKLIST")) {  // one pass with the tile in registers when the grid fits the chip
    const bool done = dt == SB_BF16 ? launch_tensorwise_coop(h, static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, q,
                                                             ldq, q_t, ldqt, state, sync, err)
                                    : launch_tensorwise_coop(h, static_cast<const float*>(x), rows, cols, ldx, q, ldq,
                                                             q_t, ldqt, state, sync, err);
    if (done) return true;
  }
  static int cap_bf16[16] = {}, cap_f32[16] = {};  // co-resident blocks per device
  int& cap = (dt == SB_BF16 ? cap_bf16 : cap_f32)[h->device & 15];
  if (cap == 0) {
    int b = 0;
    if (dt == SB_BF16)
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_quantize_tensorwise_fused<__nv_bfloat16>, 256, 0);
    else
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_quantize_tensorwise_fused<float>, 256, 0);
    cap = std::max(1, std::min(b, 4)) * h->num_sms;
  }
  const int64_t slab = std::max<int64_t>(1, 32768 / (cols * static_cast<int64_t>(dt == SB_BF16 ? 2 : 4)));
  const int64_t tasks = (rows + slab - 1) / slab + ((rows + 63) / 64) * ((cols + 63) / 64);
  const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(tasks, cap)));
  *err = cudaMemsetAsync(sync, 0, 4 * sizeof(unsigned int), h->stream);
  if (*err != cudaSuccess) return true;
  h->launches++;
  if (dt == SB_BF16)
    sb::launch_pdl(k_quantize_tensorwise_fused<__nv_bfloat16>, dim3(grid), dim3(256), 0, h->stream,
                   static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, q, ldq, q_t, ldqt, state, sync, h->d_err);
  else
    sb::launch_pdl(k_quantize_tensorwise_fused<float>, dim3(grid), dim3(256), 0, h->stream, static_cast<const float*>(x),
                   rows, cols, ldx, q, ldq, q_t, ldqt, state, sync, h->d_err);
  *err = cudaGetLastError();
  return true;
}

cudaError_t launch_absmax_rows(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                               unsigned int* words) {
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  h->launches++;
  if (dt == SB_BF16)
    k_absmax_rows<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, words);
  else
    k_absmax_rows<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, words);
  return cudaGetLastError();
}

cudaError_t launch_absmax_columns(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                  unsigned int* words) {
  cudaError_t e = cudaMemsetAsync(words, 0, sizeof(unsigned int) * cols, h->stream);
  if (e != cudaSuccess) return e;
  const unsigned gx = static_cast<unsigned>((cols + 31) / 32);
  int64_t gy = (rows + 63) / 64;
  const int64_t cap = (static_cast<int64_t>(h->num_sms) * 8 + gx - 1) / gx;
  if (gy > cap) gy = cap;
  if (gy < 1) gy = 1;
  h->launches++;
  const dim3 grid(gx, static_cast<unsigned>(gy));
  if (dt == SB_BF16)
    k_absmax_columns<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, words);
  else
    k_absmax_columns<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, words);
  return cudaGetLastError();
}

cudaError_t launch_quantize_from_words(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                       int64_t ldx, const unsigned int* words, int per_column, int8_t* q, int64_t ldq,
                                       int8_t* q_t, int64_t ldqt, float* state) {
  const dim3 grid(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
  h->launches++;
  if (dt == SB_BF16)
    k_quantize_from_words<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, words,
                                                       per_column, q, ldq, q_t, ldqt, state, h->d_err);
  else
    k_quantize_from_words<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, words,
                                                       per_column, q, ldq, q_t, ldqt, state, h->d_err);
  return cudaGetLastError();
}

cudaError_t launch_dequantize(sb_handle h, const int8_t* q, int64_t rows, int64_t cols, int64_t ldq,
                              const float* state, int axis, void* y, sb_dtype ydt, int64_t ldy) {
  const unsigned grid = grid_for(rows * cols, 256 * 4, h->num_sms);
  h->launches++;
  if (ydt == SB_BF16)
    k_dequantize<<<grid, 256, 0, h->stream>>>(q, rows, cols, ldq, state, axis, static_cast<__nv_bfloat16*>(y), ldy);
  else
    k_dequantize<<<grid, 256, 0, h->stream>>>(q, rows, cols, ldq, state, axis, static_cast<float*>(y), ldy);
  return cudaGetLastError();
}

// Fast fp8 paths (16-byte vectorisable x, q): row axis fused in one register-resident pass
// (returns true, nothing else to launch); tensor / column axis after their absmax kernel.
// Returns false when the generic kernels must run.
bool launch_quantize_fp8_fast(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                              int fmt, int axis, const unsigned int* words, uint8_t* q, int64_t ldq, float* state,
                              bool row_fused, cudaError_t* err) {
  const int vec = dt == SB_BF16 ? 8 : 4;
  if (cols % vec || ldx % vec || ldq % vec || !sb::aligned(x, 16) || !sb::aligned(q, vec) || rows <= 0 || cols <= 0)
    return false;
  if (row_fused) {
    if (axis != SB_AXIS_ROW) return false;
    h->launches++;
    const bool ok = dt == SB_BF16 ? fp8_rows_reg(h, static_cast<const __nv_bfloat16*>(x), rows,
                                                 static_cast<int>(cols / vec), ldx, fmt, q, ldq, state)
                                  : fp8_rows_reg(h, static_cast<const float*>(x), rows, static_cast<int>(cols / vec),
                                                 ldx, fmt, q, ldq, state);
    if (!ok) {
      h->launches--;
      return false;
    }
    *err = cudaGetLastError();
    return true;
  }
  if (axis == SB_AXIS_ROW) return false;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(rows, static_cast<int64_t>(h->num_sms) * 8));
  h->launches++;
  if (dt == SB_BF16)
    k_quantize_fp8_vec<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, fmt, axis,
                                                    words, q, ldq, state, h->d_err);
  else
    k_quantize_fp8_vec<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, fmt, axis, words, q,
                                                    ldq, state, h->d_err);
  *err = cudaGetLastError();
  return true;
}

cudaError_t launch_quantize_fp8(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                int fmt, int axis, const unsigned int* words, uint8_t* q, int64_t ldq, float* state) {
  const unsigned grid = grid_for(rows * cols, 256 * 4, h->num_sms);
  h->launches++;
  if (dt == SB_BF16)
    k_quantize_fp8<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), rows, cols, ldx, fmt, axis,
                                                words, q, ldq, state, h->d_err);
  else
    k_quantize_fp8<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), rows, cols, ldx, fmt, axis, words, q,
                                                ldq, state, h->d_err);
  return cudaGetLastError();
}

cudaError_t launch_dequantize_fp8(sb_handle h, const uint8_t* q, int64_t rows, int64_t cols, int64_t ldq, int fmt,
                                  const float* state, int axis, void* y, sb_dtype ydt, int64_t ldy) {
  const unsigned grid = grid_for(rows * cols, 256 * 4, h->num_sms);
  h->launches++;
  if (ydt == SB_BF16)
    k_dequantize_fp8<<<grid, 256, 0, h->stream>>>(q, rows, cols, ldq, fmt, state, axis,
                                                  static_cast<__nv_bfloat16*>(y), ldy);
  else
    k_dequantize_fp8<<<grid, 256, 0, h->stream>>>(q, rows, cols, ldq, fmt, state, axis, static_cast<float*>(y), ldy);
  return cudaGetLastError();
}

cudaError_t launch_fp8_cast(sb_handle h, const float* x, int64_t n, int fmt, float* y) {
  const unsigned grid = grid_for(n, 256 * 4, h->num_sms);
  h->launches++;
  k_fp8_cast<<<grid, 256, 0, h->stream>>>(x, n, fmt, y, h->d_err);
  return cudaGetLastError();
}

template <typename T>
__global__ void k_add_bias(T* __restrict__ y, int64_t rows, int64_t cols, const float* __restrict__ bias) {
  const int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = static_cast<float>(y[i]);
    y[i] = static_cast<T>(__fadd_rn(v, bias[i % cols]));
  }
}

template <typename T>
__global__ void k_add_residual(T* __restrict__ y, int64_t n, const T* __restrict__ r) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = static_cast<T>(__fadd_rn(static_cast<float>(y[i]), static_cast<float>(r[i])));
}

cudaError_t launch_add_residual(sb_handle h, void* y, sb_dtype dt, int64_t rows, int64_t cols, const void* resid) {
  const int64_t n = rows * cols;
  const unsigned grid = grid_for(n, 256 * 4, h->num_sms);
  h->launches++;
  if (dt == SB_F32)
    k_add_residual<<<grid, 256, 0, h->stream>>>(static_cast<float*>(y), n, static_cast<const float*>(resid));
  else if (dt == SB_BF16)
    k_add_residual<<<grid, 256, 0, h->stream>>>(static_cast<__nv_bfloat16*>(y), n,
                                                static_cast<const __nv_bfloat16*>(resid));
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_add_bias(sb_handle h, void* y, sb_dtype dt, int64_t rows, int64_t cols, const float* bias) {
  const unsigned grid = grid_for(rows * cols, 256 * 4, h->num_sms);
  h->launches++;
  if (dt == SB_F32)
    k_add_bias<<<grid, 256, 0, h->stream>>>(static_cast<float*>(y), rows, cols, bias);
  else if (dt == SB_BF16)
    k_add_bias<<<grid, 256, 0, h->stream>>>(static_cast<__nv_bfloat16*>(y), rows, cols, bias);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_ln_quantize_rowwise(sb_handle h, const void* x, int64_t rows, int64_t cols, const float* gamma,
                                       const float* beta, float eps, void* out, int8_t* q, float* state, float* mean,
                                       float* rstd) {
  using bf = __nv_bfloat16;
  if (cols % 8 || !sb::aligned(x, 16) || !sb::aligned(out, 16) || !sb::aligned(q, 8) || !sb::aligned(gamma, 16) ||
      !sb::aligned(beta, 16))
    return cudaErrorNotSupported;
  const int nvec = static_cast<int>(cols / 8);
  const bf* X = static_cast<const bf*>(x);
  bf* O = static_cast<bf*>(out);
  switch ((nvec + 31) / 32) {
    case 1: launch_ln_rows<1>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 2: launch_ln_rows<2>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 3: launch_ln_rows<3>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 4: launch_ln_rows<4>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 5: launch_ln_rows<5>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 6: launch_ln_rows<6>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    case 7:
    case 8: launch_ln_rows<8>(h, X, rows, nvec, gamma, beta, eps, O, q, state, mean, rstd); break;
    default: return cudaErrorNotSupported;  // rows longer than 2048: not fused
  }
  return cudaGetLastError();
}

// Blocks the LayerNorm backward launches (its partial buffer holds 2 * cols floats per block).
int64_t ln_backward_blocks(sb_handle h) { return static_cast<int64_t>(h->num_sms) * 2; }  // 2 blocks of 8 warps / SM

cudaError_t launch_ln_backward(sb_handle h, const void* dh, const void* x, int64_t rows, int64_t cols,
                               const float* mean, const float* rstd, const float* gamma, void* dx, float* dgamma,
                               float* dbeta, float* part) {
  using bf = __nv_bfloat16;
  if (cols % 8 || cols > 1280 || !sb::aligned(dh, 16) || !sb::aligned(x, 16) || !sb::aligned(dx, 16) ||
      !sb::aligned(part, 16))
    return cudaErrorNotSupported;
  const int nvec = static_cast<int>(cols / 8);
  const int64_t blocks = ln_backward_blocks(h);
  const bf* D = static_cast<const bf*>(dh);
  const bf* X = static_cast<const bf*>(x);
  bf* O = static_cast<bf*>(dx);
  const size_t smem = static_cast<size_t>(8) * nvec * (1 + 2 * 8) * sizeof(float);  // gamma + 8 warps x 2
  h->launches++;
  switch ((nvec + 31) / 32) {
    case 1: launch_ln_bwd<1>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part); break;
    case 2: launch_ln_bwd<2>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part); break;
    case 3: launch_ln_bwd<3>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part); break;
    case 4: launch_ln_bwd<4>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part); break;
    default: launch_ln_bwd<5>(h, blocks, smem, D, X, rows, nvec, mean, rstd, gamma, O, part); break;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  h->launches++;
  k_ln_bwd_reduce<<<static_cast<unsigned>((2 * cols + 31) / 32), 256, 0, h->stream>>>(part, blocks, static_cast<int>(cols),
                                                                                        dgamma, dbeta);
  return cudaGetLastError();
}

cudaError_t build_gelu_lut(sb_handle h) {
  if (h->gelu_lut) return cudaSuccess;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, static_cast<size_t>(kFwdEntries) * 2 + static_cast<size_t>(kLutEntries) * 4);
  if (e != cudaSuccess) return e;
  k_build_gelu_lut<<<64, 256>>>(static_cast<__nv_bfloat16*>(p),
                               reinterpret_cast<float*>(static_cast<uint8_t*>(p) + static_cast<size_t>(kFwdEntries) * 2));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(p);
    return e;
  }
  h->gelu_lut = p;
  return cudaSuccess;
}

cudaError_t launch_heads_pack_quantize(sb_handle h, const void* const* src, const int64_t* strides, int64_t B,
                                       int64_t S, int H, int Dh, void* g, int8_t* const* q, float* const* st) {
  const int D = H * Dh;
  if (Dh % 8 || D > 2048 || B <= 0 || S <= 0 || !sb::aligned(g, 16)) return cudaErrorNotSupported;
  HeadsSrc hs{};
  for (int i = 0; i < 3; ++i) {
    hs.p[i] = static_cast<const __nv_bfloat16*>(src[i]);
    hs.sb[i] = strides[3 * i];
    hs.sh[i] = strides[3 * i + 1];
    hs.ss[i] = strides[3 * i + 2];
    hs.q[i] = q[i];
    hs.st[i] = st[i];
    if (!sb::aligned(src[i], 16) || hs.sb[i] % 8 || hs.sh[i] % 8 || hs.ss[i] % 8 || !sb::aligned(q[i], 8))
      return cudaErrorNotSupported;
  }
  const int64_t T = B * S;
  const int vpl = (D / 8 + 31) / 32;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((3 * T + 7) / 8, 8LL * h->num_sms));
  h->launches++;
  switch (vpl) {
    case 1: k_heads_pack_quantize<1><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 2: k_heads_pack_quantize<2><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 3: k_heads_pack_quantize<3><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 4: k_heads_pack_quantize<4><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 5: k_heads_pack_quantize<5><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 6: k_heads_pack_quantize<6><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    case 7: k_heads_pack_quantize<7><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
    default: k_heads_pack_quantize<8><<<grid, 256, 0, h->stream>>>(hs, S, H, Dh, T, static_cast<__nv_bfloat16*>(g), h->d_err); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_act_quantize_rowwise(sb_handle h, int mode, const void* a, const void* b, int64_t rows, int64_t cols,
                                        void* act, int8_t* q, float* state) {
  using bf = __nv_bfloat16;
  const bf* A = static_cast<const bf*>(a);
  const bf* B = static_cast<const bf*>(b);
  bf* O = static_cast<bf*>(act);
  const bool vec_ok = h->gelu_lut && cols % 8 == 0 && sb::aligned(a, 16) && (mode == 0 || sb::aligned(b, 16)) &&
                      sb::aligned(act, 16) && sb::aligned(q, 8) && cols / 8 < (1 << 30);
  if (vec_ok) {
    const int nvec = static_cast<int>(cols / 8);
    const char* ce = getenv("SB_ACT_CH");  // measurement switch: vectors per lane per step
    const int ch = ce ? atoi(ce) : 2;
    if (mode == 0)
      return ch == 4 ? launch_act_rows<0, 4>(h, A, B, rows, nvec, O, q, state)
                     : ch == 1 ? launch_act_rows<0, 1>(h, A, B, rows, nvec, O, q, state)
                               : launch_act_rows<0, 2>(h, A, B, rows, nvec, O, q, state);
    return ch == 4 ? launch_act_rows<1, 4>(h, A, B, rows, nvec, O, q, state)
                   : ch == 1 ? launch_act_rows<1, 1>(h, A, B, rows, nvec, O, q, state)
                             : launch_act_rows<1, 2>(h, A, B, rows, nvec, O, q, state);
  }
  const unsigned grid = grid_for(rows * cols, 256 * 4, h->num_sms);
  h->launches++;
  if (mode == 0)
    k_act_elementwise<0><<<grid, 256, 0, h->stream>>>(A, B, rows * cols, O);
  else
    k_act_elementwise<1><<<grid, 256, 0, h->stream>>>(A, B, rows * cols, O);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_quantize_rowwise(h, act, SB_BF16, rows, cols, cols, q, cols, state);
}

cudaError_t launch_convert(sb_handle h, const void* x, sb_dtype xdt, void* y, sb_dtype ydt, int64_t n) {
  const unsigned grid = grid_for(n, 256 * 4, h->num_sms);
  h->launches++;
  if (xdt == SB_F32 && ydt == SB_BF16)
    k_convert<<<grid, 256, 0, h->stream>>>(static_cast<const float*>(x), static_cast<__nv_bfloat16*>(y), n);
  else if (xdt == SB_BF16 && ydt == SB_F32)
    k_convert<<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(x), static_cast<float*>(y), n);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace sb
