// optim.cu — K7: multi-tensor StableAdamW (optimizer.cpp:102-172), HBM-bound.
//
// Per tensor the reference is a three-pass loop: moments (:142-146), RMS from the
// UPDATED second moment (:148-157), then the parameter update (:162-167), so the RMS
// couples every element before any theta can move. On B200 that is two kernels per
// group of tensors:
//   phase 1  read g, v, u; write v, u; per-block sum of g^2 / max(u, eps^2) (fp64, fixed
//            tree order) -> partials[block]
//   phase 2  per block: reduce its tensor's partials in block order -> RMS, eta; read
//            theta (+ v, u from L2: the group is sized to keep v,u L2-resident), write theta
// Algorithmic traffic 28 B/param (read theta, g, v, u; write theta, v, u). Element math is
// fp64 with explicitly rounded operations (__dmul_rn/__dadd_rn/...), mirroring the
// reference's double arithmetic under -ffp-contract=off, so v/u/theta are bit-identical
// whenever eta does not depend on the reduction order.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cuda_bf16.h>

#include "sb_internal.h"

namespace {

// 128-thread blocks, 9 per SM (56 registers, a 24-byte spill): 6.27 ms per 1e9-param step vs
// 6.44 (8 per SM, 64 regs), 6.59 (256 x 4), 6.80 (512 x 2), 7.0 (11-12 per SM: heavy spills)
constexpr int kThreads = 128;
constexpr int kPerThread = 16;
constexpr int kChunk = kThreads * kPerThread;  // elements per block task
constexpr int kMaxGroup = 256;                 // tensors per launch (kernel parameters <= 32 KB)
constexpr int kVecPerIter = 1;                 // float4 groups loaded per inner iteration (register budget)

struct TensorDesc {
  float* theta;
  const float* grad;
  float* v;
  float* u;
  int64_t numel;
  int64_t block0;  // first chunk of this tensor in the group (= index of its first partial)
  int64_t nblocks;
  int64_t task0;   // first phase-1 task (tasks [task0, task0 + nblocks))
  int64_t task2;   // first phase-2 task
  int32_t index;   // position in the caller's tensor list (rms/eta outputs)
  int32_t vec;     // all four arrays 16-byte aligned and numel % 4 == 0: float4 path
  __nv_bfloat16* shadow;  // optional: bf16(theta') for the next forward (sb_adamw_extras)
  unsigned int* word;     // optional: max |bf16(theta')| as fp32 bits
  double numel_total;     // elements of the whole tensor (RMS denominator): numel, or the
                          // full tensor's count when this is one rank's shard (ZeRO-1)
};

struct Group {
  TensorDesc t[kMaxGroup];
  // task segments in fetch order: phase 1 of tensor k+1 precedes phase 2 of tensor k, so a
  // phase-2 task never waits on chunks still in flight (seg = 2*k + phase)
  int64_t seg_start[2 * kMaxGroup];
  int16_t seg_id[2 * kMaxGroup];
  int count;
  int nseg;  // segments in seg_start / seg_id (2 * count fused, count per ZeRO-1 phase)
  int64_t total_blocks;
  int64_t total_tasks;
};

struct Coeffs {
  double b1, omb1, b2, omb2;  // debiased decay rates and their complements (host-computed)
  double floor_;              // eps^2
  double eps, alpha, wd;
  int32_t update_clip;
  // filter_nonfinite's unscaling (optimizer.cpp:91-92), g' = f32(double(g) / scale):
  // 0 none, 1 scale is a power of two (then g' = g * fl(1/scale) in fp32, exact and identical),
  // 2 general (fp64 division)
  int32_t scale_mode;
  float inv_scale_f;
  double scale;
  const int32_t* skipped;  // per caller tensor index: 1 = leave this tensor untouched (or null)
};

// The gradient the update sees: unscaled (EX), then the in-step clip factor.
template <bool EX>
__device__ __forceinline__ double grad_in(const Coeffs& c, float g, double clip) {
  if (EX && c.scale_mode == 1) g = __fmul_rn(g, c.inv_scale_f);
  if (EX && c.scale_mode == 2) g = __double2float_rn(__ddiv_rn(static_cast<double>(g), c.scale));
  return clip == 1.0 ? static_cast<double>(g) : __dmul_rn(static_cast<double>(g), clip);
}
__device__ __forceinline__ uint32_t bf16_abs_bits(__nv_bfloat16 b) {  // as fp32 bits (quantize.cu abs_bits)
  return (static_cast<uint32_t>(__bfloat16_as_ushort(b)) & 0x7fffu) << 16;
}

template <typename F>
__device__ __forceinline__ int find_by(const Group& g, F key, int64_t x) {
  int lo = 0, hi = g.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (key(g.t[mid]) <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int find_tensor(const Group& g, int64_t blk) {
  return find_by(g, [](const TensorDesc& d) { return d.block0; }, blk);
}

// Deterministic block sum: per-warp xor-tree, then warp 0 over the 8 warp sums.
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) s = __dadd_rn(s, red[i]);
  __syncthreads();  // red reusable
  return s;
}

__device__ __forceinline__ uint32_t ld_acquire(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The kernel was bound by the XU pipe (ncu: 93% of its realtime peak): the f32 <-> f64
// conversions (F2F) and the MUFU seeds of DDIV / DSQRT run there, while the fp64 FMA pipe sat
// at ~35% and DRAM at 67%. Taking the RMS term's division off the XU pipe (rcp_nr) took the
// 1e9-parameter step from 6.27 to 5.85 ms. (Exact f32 -> f64 conversion on the integer pipes
// instead of F2F was slower: 7.3 ms.)
// 1 / x for the RMS terms only (they are summed, and RMS is compared to 1e-12): an
// integer-seeded reciprocal (relative error <= 1/8) refined by four Newton steps on the fp64 FMA
// pipe (error squares each step: < 2^-53 after four) — no MUFU on the XU pipe. x >= eps^2 > 0.
__device__ __forceinline__ double rcp_nr(double x) {
  double r = __longlong_as_double(0x7FDE623822FC16E6LL - __double_as_longlong(x));
#pragma unroll
  for (int i = 0; i < 4; ++i) r = __fma_rn(r, __fma_rn(-x, r, 1.0), r);
  return r;
}
// Moments of one element (optimizer.cpp:142-146) and its RMS term g^2 / max(u, eps^2) (:148-157).
__device__ __forceinline__ double moments(const Coeffs& c, double g, float& v, float& u) {
  v = __double2float_rn(__dadd_rn(__dmul_rn(c.b1, static_cast<double>(v)), __dmul_rn(c.omb1, g)));
  u = __double2float_rn(__dadd_rn(__dmul_rn(c.b2, static_cast<double>(u)), __dmul_rn(__dmul_rn(c.omb2, g), g)));
  const double ud = static_cast<double>(u);
  return __dmul_rn(__dmul_rn(g, g), rcp_nr(ud > c.floor_ ? ud : c.floor_));
}
// Parameter update of one element (optimizer.cpp:162-167), correctly rounded throughout (DSQRT,
// DDIV). A certified MUFU-free variant (integer-seeded Newton sqrt / reciprocal on the FMA pipe,
// integer rounding to f32 when r is provably far from a rounding midpoint, exact fallback
// otherwise) was bit-identical but slower, 6.67 vs 5.85 ms per 1e9 parameters: with the RMS
// term's MUFU gone the FMA pipe, not the XU pipe, is the next limit.
__device__ __forceinline__ float update(const Coeffs& c, double eta, double eta_wd, float th_f, float v, float u) {
  const double th = static_cast<double>(th_f);
  const double upd = __ddiv_rn(static_cast<double>(v), __dadd_rn(__dsqrt_rn(static_cast<double>(u)), c.eps));
  return __double2float_rn(__dsub_rn(__dsub_rn(th, __dmul_rn(eta_wd, th)), __dmul_rn(eta, upd)));
}

// Phase-1 work on chunk `blk` of tensor d: moments + partial RMS sum (fixed order).
template <bool EX>
__device__ __forceinline__ double phase1_chunk(const TensorDesc& d, const Coeffs& c, double clip, int64_t blk) {
  const int64_t base = blk * kChunk;
  double acc = 0.0;
  if (d.vec) {
    // thread owns 4 float4 groups: elements base + (e*256 + tid)*4 .. +3 (coalesced 16 B),
    // loaded two groups at a time (register budget for 2 blocks / SM)
#pragma unroll
    for (int hh = 0; hh < kPerThread / 4 / kVecPerIter; ++hh) {
      float4 gv[kVecPerIter], vv[kVecPerIter], uv[kVecPerIter];
#pragma unroll
      for (int e = 0; e < kVecPerIter; ++e) {
        const int64_t i = base + (static_cast<int64_t>(kVecPerIter * hh + e) * kThreads + threadIdx.x) * 4;
        if (i < d.numel) {
          gv[e] = __ldcs(reinterpret_cast<const float4*>(d.grad + i));
          vv[e] = __ldcg(reinterpret_cast<const float4*>(d.v + i));
          uv[e] = __ldcg(reinterpret_cast<const float4*>(d.u + i));
        }
      }
#pragma unroll
      for (int e = 0; e < kVecPerIter; ++e) {
        const int64_t i = base + (static_cast<int64_t>(kVecPerIter * hh + e) * kThreads + threadIdx.x) * 4;
        if (i < d.numel) {
          const float ga[4] = {gv[e].x, gv[e].y, gv[e].z, gv[e].w};
          float va[4] = {vv[e].x, vv[e].y, vv[e].z, vv[e].w};
          float ua[4] = {uv[e].x, uv[e].y, uv[e].z, uv[e].w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc = __dadd_rn(acc, moments(c, grad_in<EX>(c, ga[k], clip), va[k], ua[k]));
          }
          *reinterpret_cast<float4*>(d.v + i) = make_float4(va[0], va[1], va[2], va[3]);
          *reinterpret_cast<float4*>(d.u + i) = make_float4(ua[0], ua[1], ua[2], ua[3]);
        }
      }
    }
  } else {
    for (int e = 0; e < kPerThread; ++e) {
      const int64_t i = base + e * kThreads + threadIdx.x;
      if (i < d.numel) {
        float v = d.v[i], u = d.u[i];
        acc = __dadd_rn(acc, moments(c, grad_in<EX>(c, d.grad[i], clip), v, u));
        d.v[i] = v;
        d.u[i] = u;
      }
    }
  }
  return acc;
}

// Phase-2 work on chunk `blk`: theta update (kept as is when `keep`: a skipped tensor), plus with
// EX the bf16 shadow copy; returns this thread's max |bf16(theta')| as fp32 bits (0 without EX).
template <bool EX>
__device__ __forceinline__ uint32_t phase2_chunk(const TensorDesc& d, const Coeffs& c, double eta, int64_t blk,
                                                 bool keep) {
  const double eta_wd = __dmul_rn(eta, c.wd);
  const int64_t base = blk * kChunk;
  uint32_t amax = 0;
  if (d.vec) {
#pragma unroll
    for (int hh = 0; hh < kPerThread / 4 / kVecPerIter; ++hh) {
      float4 tv[kVecPerIter], vv[kVecPerIter], uv[kVecPerIter];
#pragma unroll
      for (int e = 0; e < kVecPerIter; ++e) {
        const int64_t i = base + (static_cast<int64_t>(kVecPerIter * hh + e) * kThreads + threadIdx.x) * 4;
        if (i < d.numel) {
          tv[e] = __ldcs(reinterpret_cast<const float4*>(d.theta + i));
          if (!EX || !keep) {
            vv[e] = __ldcs(reinterpret_cast<const float4*>(d.v + i));
            uv[e] = __ldcs(reinterpret_cast<const float4*>(d.u + i));
          }
        }
      }
#pragma unroll
      for (int e = 0; e < kVecPerIter; ++e) {
        const int64_t i = base + (static_cast<int64_t>(kVecPerIter * hh + e) * kThreads + threadIdx.x) * 4;
        if (i < d.numel) {
          float4 o = tv[e];
          if (!EX || !keep) {
            o.x = update(c, eta, eta_wd, tv[e].x, vv[e].x, uv[e].x);
            o.y = update(c, eta, eta_wd, tv[e].y, vv[e].y, uv[e].y);
            o.z = update(c, eta, eta_wd, tv[e].z, vv[e].z, uv[e].z);
            o.w = update(c, eta, eta_wd, tv[e].w, vv[e].w, uv[e].w);
            __stcs(reinterpret_cast<float4*>(d.theta + i), o);
          }
          if (EX && d.shadow != nullptr) {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
            amax = max(max(amax, max(bf16_abs_bits(lo.x), bf16_abs_bits(lo.y))),
                       max(bf16_abs_bits(hi.x), bf16_abs_bits(hi.y)));
            uint2 pk;
            pk.x = *reinterpret_cast<const uint32_t*>(&lo);
            pk.y = *reinterpret_cast<const uint32_t*>(&hi);
            *reinterpret_cast<uint2*>(d.shadow + i) = pk;
          }
        }
      }
    }
  } else {
    for (int e = 0; e < kPerThread; ++e) {
      const int64_t i = base + e * kThreads + threadIdx.x;
      if (i < d.numel) {
        const float o = (EX && keep) ? d.theta[i] : update(c, eta, eta_wd, d.theta[i], d.v[i], d.u[i]);
        if (!EX || !keep) d.theta[i] = o;
        if (EX && d.shadow != nullptr) {
          const __nv_bfloat16 b = __float2bfloat16_rn(o);
          d.shadow[i] = b;
          amax = max(amax, bf16_abs_bits(b));
        }
      }
    }
  }
  return amax;
}

// Persistent multi-tensor StableAdamW. Tasks, fetched in order from an atomic counter:
// phase-1 chunks of tensor k+1 precede phase-2 chunks of tensor k. The block that completes
// a tensor's last phase-1 chunk reduces the tensor's partials in a fixed order (same sum
// whichever block it is), computes RMS and eta once and publishes eta; a phase-2 chunk waits
// for that flag (every phase-1 chunk of its tensor was fetched before it, by running blocks:
// no deadlock) and updates theta while v, u of the tensor are still in L2. No launch
// boundary between tensors: phase 1 of tensor k+1 overlaps the tail of tensor k.
// sync[0] = task counter, sync[1 + 2k] = finished phase-1 chunks of group tensor k,
// sync[2 + 2k] = its eta-ready flag (zeroed by the launcher); eta_buf[k] = its eta.
__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// MODE 0: the fused step above. MODE 1 (ZeRO-1 phase 1): phase-1 tasks only; the tensor's fixed-
// order sum of g^2 / max(u, eps^2) over this rank's shard goes to eta_buf[index] (the caller sums
// it over ranks). MODE 2 (ZeRO-1 phase 2): phase-2 tasks only; eta_buf[index] holds the sum over
// every rank's shard, from which each task forms RMS over the whole tensor (numel_total) and eta.
template <bool EX, int MODE = 0>
__global__ void __launch_bounds__(kThreads, EX ? 8 : 9) k_adamw_persistent(const __grid_constant__ Group grp, Coeffs c,
                                                               const double* __restrict__ clip_ptr,
                                                               double* __restrict__ partials,
                                                               unsigned int* __restrict__ sync,
                                                               double* __restrict__ eta_buf, double* rms_out,
                                                               double* eta_out) {
  __shared__ double red[kThreads / 32];
  __shared__ int64_t s_task;
  __shared__ double s_eta;
  __shared__ int s_last;
  const double clip = clip_ptr ? *clip_ptr : 1.0;
  // The next task id is claimed when the current one starts, so the ~1 us atomic round trip
  // overlaps the chunk's loads instead of stalling the whole block between chunks (6.71 ->
  // 6.59 ms per 1e9-param step). A block holds at most one claimed-but-unstarted id, larger
  // than its current one: the lowest unfinished id is always some block's current task, so
  // the no-deadlock argument below still holds. (Fewer barriers per chunk -- warp 0 alone
  // finishing the block sum -- measured slower: 7.02 ms, registers spill at 64.)
  if (threadIdx.x == 0) s_task = atomicAdd(sync, 1u);
  __syncthreads();
  for (;;) {
    const int64_t task = s_task;
    __syncthreads();
    if (task >= grp.total_tasks) break;
    unsigned int next = 0;
    if (threadIdx.x == 0) next = atomicAdd(sync, 1u);
    int lo = 0, hi = grp.nseg - 1;  // segment containing `task`
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (grp.seg_start[mid] <= task) lo = mid;
      else hi = mid - 1;
    }
    const int seg = grp.seg_id[lo];
    const int ti = seg >> 1;
    const TensorDesc& d = grp.t[ti];
    const int64_t local = (seg & 1) ? d.nblocks + (task - d.task2) : task - d.task0;
    const bool skip = EX && c.skipped != nullptr && c.skipped[d.index] != 0;
    if (MODE == 2) {
      if (threadIdx.x == 0) {
        const double rms = __dsqrt_rn(__ddiv_rn(__ldcg(eta_buf + d.index), d.numel_total));
        const double eta = c.update_clip ? __ddiv_rn(c.alpha, rms > 1.0 ? rms : 1.0) : c.alpha;
        s_eta = eta;
        if (local == d.nblocks) {
          if (rms_out) rms_out[d.index] = rms;
          if (eta_out) eta_out[d.index] = eta;
        }
      }
      __syncthreads();
      const uint32_t m = phase2_chunk<EX>(d, c, s_eta, local - d.nblocks, false);
      if (EX && d.word != nullptr) {
        const uint32_t wm = __reduce_max_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0 && wm != 0u) atomicMax(d.word, wm);
      }
    } else if (local < d.nblocks) {
      const double s = block_sum(skip ? 0.0 : phase1_chunk<EX>(d, c, clip, local), red);
      if (threadIdx.x == 0) {
        partials[d.block0 + local] = s;
        __threadfence();
        s_last = atomicAdd(sync + 1 + 2 * ti, 1u) == static_cast<unsigned int>(d.nblocks - 1);
      }
      __syncthreads();
      if (s_last) {
        // the block that finished the tensor's last chunk reduces its partials in a fixed
        // order (thread-strided, then the block tree: the same sum whichever block does it),
        // computes RMS and eta once and publishes eta for the phase-2 chunks
        __threadfence();
        double sum = 0.0;
        for (int64_t j = threadIdx.x; j < d.nblocks; j += kThreads) sum = __dadd_rn(sum, __ldcg(partials + d.block0 + j));
        const double tot = block_sum(sum, red);
        if (MODE == 1) {
          if (threadIdx.x == 0) eta_buf[d.index] = tot;
        } else if (threadIdx.x == 0) {
          double rms = __dsqrt_rn(__ddiv_rn(tot, static_cast<double>(d.numel)));
          double eta = c.update_clip ? __ddiv_rn(c.alpha, rms > 1.0 ? rms : 1.0) : c.alpha;
          if (skip) {  // trainer.cpp:140-143: a skipped tensor reports rms = NaN
            rms = __longlong_as_double(0x7ff8000000000000LL);
            eta = 0.0;
          }
          if (EX && d.word != nullptr) *d.word = 0u;  // the phase-2 chunks max into it after the flag
          eta_buf[ti] = eta;
          if (rms_out) rms_out[d.index] = rms;
          if (eta_out) eta_out[d.index] = eta;
          __threadfence();
          st_release(sync + 2 + 2 * ti, 1u);
        }
      }
    } else {
      if (threadIdx.x == 0) {
        while (ld_acquire(sync + 2 + 2 * ti) == 0u) __nanosleep(100);
        s_eta = __ldcg(eta_buf + ti);
      }
      __syncthreads();
      const uint32_t m = phase2_chunk<EX>(d, c, s_eta, local - d.nblocks, skip);
      if (EX && d.word != nullptr) {
        const uint32_t wm = __reduce_max_sync(0xffffffffu, m);
        if ((threadIdx.x & 31) == 0 && wm != 0u) atomicMax(d.word, wm);
      }
    }
    if (threadIdx.x == 0) s_task = next;
    __syncthreads();
  }
}

// Empty tensors have no chunks: the reference still reports them, with rms = sqrt(0 / 0) = NaN
// and eta = alpha / max(1, NaN) = alpha (std::max returns its first argument when the
// comparison is false), optimizer.cpp:148-160.
struct EmptyList {
  int32_t index[64];
  int count;
};
__global__ void k_empty_infos(const __grid_constant__ EmptyList e, double alpha, double* rms_out, double* eta_out) {
  const int i = threadIdx.x;
  if (i >= e.count) return;
  if (rms_out) rms_out[e.index[i]] = __longlong_as_double(0x7ff8000000000000LL);
  if (eta_out) eta_out[e.index[i]] = alpha;
}

// Statistics pass of sb_stableadamw_step_ex (one read of g, before any state changes): per
// chunk the unscaled gradient's non-finite flag, |g'| max and sum of g'^2; the block that
// finishes a tensor's last chunk sums the tensor's partials in a fixed order into tensor_ss.
// counts[k] (zeroed) counts finished chunks of group tensor k.
__global__ void __launch_bounds__(kThreads) k_gradstats(const __grid_constant__ Group grp, Coeffs c,
                                                        double* __restrict__ partials, int64_t offset,
                                                        unsigned int* __restrict__ counts, double* __restrict__ tensor_ss,
                                                        int32_t* __restrict__ skipped, unsigned int* __restrict__ amax_bits) {
  __shared__ double red[kThreads / 32];
  __shared__ int s_last;
  const int64_t gblk = offset + blockIdx.x;
  const int ti = find_tensor(grp, gblk);
  const TensorDesc& d = grp.t[ti];
  const int64_t base = (gblk - d.block0) * kChunk;
  double acc = 0.0;
  uint32_t amax = 0, bad = 0;
  for (int e = 0; e < kPerThread; ++e) {
    const int64_t i = base + e * kThreads + threadIdx.x;
    if (i < d.numel) {
      const double gd = grad_in<true>(c, d.grad[i], 1.0);
      const uint32_t ab = __float_as_uint(static_cast<float>(gd)) & 0x7fffffffu;
      bad |= ab >= 0x7f800000u;                 // inf or NaN (optimizer.cpp:94)
      if (ab <= 0x7f800000u) amax = max(amax, ab);  // NaN never wins (Matrix::abs_max, matrix.cpp:31-35)
      acc = __dadd_rn(acc, __dmul_rn(gd, gd));
    }
  }
  amax = __reduce_max_sync(0xffffffffu, amax);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (amax_bits != nullptr && amax != 0u) atomicMax(amax_bits + d.index, amax);
    if (bad) atomicOr(reinterpret_cast<unsigned int*>(skipped) + d.index, 1u);
  }
  const double sblk = block_sum(acc, red);
  if (threadIdx.x == 0) {
    partials[gblk] = sblk;
    __threadfence();
    s_last = atomicAdd(counts + ti, 1u) == static_cast<unsigned int>(d.nblocks - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double sum = 0.0;
    for (int64_t j = threadIdx.x; j < d.nblocks; j += kThreads) sum = __dadd_rn(sum, __ldcg(partials + d.block0 + j));
    const double tot = block_sum(sum, red);
    if (threadIdx.x == 0) tensor_ss[d.index] = tot;
  }
}

// After the statistics pass: LossScaler::per_tensor_skip == 0 turns one skip into all
// (optimizer.cpp:96-99); kGradClip's factor from the applied tensors' sums, in tensor order
// (optimizer.cpp:121-131).
__global__ void k_gradstats_final(int n, int per_tensor_skip, const double* __restrict__ tensor_ss,
                                  int32_t* __restrict__ skipped, int grad_clip, double max_norm, double* clip) {
  __shared__ double red[kThreads / 32];
  __shared__ int s_any;
  if (threadIdx.x == 0) s_any = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kThreads)
    if (skipped[i]) s_any = 1;
  __syncthreads();
  if (!per_tensor_skip && s_any)
    for (int i = threadIdx.x; i < n; i += kThreads) skipped[i] = 1;
  __syncthreads();
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads)
    if (!skipped[i]) s = __dadd_rn(s, tensor_ss[i]);
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0 && clip != nullptr) {
    const double norm = __dsqrt_rn(tot);
    *clip = (grad_clip && norm > max_norm) ? __ddiv_rn(max_norm, norm) : 1.0;
  }
}

double debias(double beta, int64_t t) {  // optimizer.cpp:63-68
  if (beta == 0.0) return 0.0;
  const double num = 1.0 - std::pow(beta, static_cast<double>(t - 1));
  const double den = 1.0 - std::pow(beta, static_cast<double>(t));
  return beta * num / den;
}

double beta2_warmup(int64_t t, double lambda) {  // optimizer.cpp:44-49
  const double b = 1.0 - std::pow(static_cast<double>(t), -lambda);
  return std::min(b, std::nextafter(1.0, 0.0));
}

std::vector<Group> make_groups(const sb_adamw_tensor* ts, int n, int64_t* total_blocks, const sb_adamw_extras* ex,
                               int mode = 0, const int64_t* numel_total = nullptr) {
  std::vector<Group> groups;
  Group cur{};
  int64_t blocks_all = 0;
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  for (int i = 0; i < n; ++i) {
    const int64_t nb = (ts[i].numel + kChunk - 1) / kChunk;
    if (cur.count == kMaxGroup) {
      groups.push_back(cur);
      cur = Group{};
    }
    if (nb == 0) continue;
    TensorDesc& d = cur.t[cur.count++];
    d.theta = ts[i].theta;
    d.grad = ts[i].grad;
    d.v = ts[i].v;
    d.u = ts[i].u;
    d.numel = ts[i].numel;
    d.numel_total = static_cast<double>(numel_total ? numel_total[i] : ts[i].numel);
    d.block0 = blocks_all;  // partials are global across groups (the grad-clip pass shares them)
    d.nblocks = nb;
    d.index = i;
    d.shadow = ex && ex->shadow_bf16 ? static_cast<__nv_bfloat16*>(ex->shadow_bf16[i]) : nullptr;
    d.word = ex && ex->absmax_word ? ex->absmax_word[i] : nullptr;
    d.vec = a16(d.theta) && a16(d.grad) && a16(d.v) && a16(d.u) && (d.numel % 4 == 0) &&
            (d.shadow == nullptr || (reinterpret_cast<uintptr_t>(d.shadow) & 7u) == 0);
    cur.total_blocks += nb;
    blocks_all += nb;
  }
  if (cur.count > 0) groups.push_back(cur);
  for (Group& g : groups) {  // fetch order: p1(0), p1(1), p2(0), p1(2), p2(1), ..., p2(last)
    int64_t tk = 0;
    int ns = 0;
    auto seg = [&](int k, int phase) {
      g.seg_start[ns] = tk;
      g.seg_id[ns] = static_cast<int16_t>(2 * k + phase);
      ++ns;
      if (phase) g.t[k].task2 = tk;
      else g.t[k].task0 = tk;
      tk += g.t[k].nblocks;
    };
    if (mode == 0) {
      for (int k = 0; k < g.count; ++k) {
        seg(k, 0);
        if (k > 0) seg(k - 1, 1);
      }
      if (g.count > 0) seg(g.count - 1, 1);
    } else {  // ZeRO-1: one phase per launch
      for (int k = 0; k < g.count; ++k) seg(k, mode == 1 ? 0 : 1);
    }
    g.total_tasks = tk;
    g.nseg = ns;
  }
  *total_blocks = blocks_all;
  return groups;
}

}  // namespace

extern "C" sb_status sb_stableadamw_workspace_size(const sb_adamw_tensor* tensors, int ntensors, size_t* bytes) {
  if (!bytes || (ntensors > 0 && !tensors)) return sb::fail(SB_ERR_INVALID_ARGUMENT, "optimizer_step", "null argument");
  int64_t total = 0;
  for (int i = 0; i < ntensors; ++i) total += (tensors[i].numel + kChunk - 1) / kChunk;
  // partials (one double per chunk), the grad-clip factor, eta per group tensor, per caller
  // tensor the statistics pass's sum of squares (double), skip flag and |g'| max word, sync
  // words (task counter + per group tensor: finished phase-1 chunks, eta-ready flag)
  *bytes = static_cast<size_t>(total + 2 + kMaxGroup + ntensors) * sizeof(double) +
           static_cast<size_t>(2 * ntensors + 2 * kMaxGroup + 2) * sizeof(unsigned int) + 64;
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_step_ex(sb_handle h, const sb_adamw_tensor* tensors, int ntensors,
                                            const sb_adamw_hparams* hp, int64_t t, const sb_adamw_extras* ex,
                                            double* rms_out, double* eta_out, void* workspace, size_t workspace_bytes) {
  const char* op = "optimizer_step";
  if (!h || !hp || (ntensors > 0 && !tensors)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null argument");
  if (t < 1) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "t must be >= 1");  // optimizer.cpp:104
  for (int i = 0; i < ntensors; ++i)  // empty tensors may come with null data pointers
    if ((tensors[i].numel != 0 && (!tensors[i].theta || !tensors[i].grad || !tensors[i].v || !tensors[i].u)) ||
        tensors[i].numel < 0)
      return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null tensor reference");  // :107-108
  if (hp->clipping == SB_CLIP_GRAD && !(hp->max_grad_norm > 0))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "grad_clip", "max_norm must be > 0");
  if (ex && !(ex->loss_scale > 0)) return sb::fail(SB_ERR_INVALID_ARGUMENT, "loss scaler", "scale must be > 0");
  size_t need = 0;
  sb_stableadamw_workspace_size(tensors, ntensors, &need);
  if (!workspace || workspace_bytes < need) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  cudaSetDevice(h->device);

  Coeffs c{};
  c.b1 = debias(hp->beta1, t);
  c.b2 = hp->beta2_warmup_lambda > 0 ? beta2_warmup(t, hp->beta2_warmup_lambda) : debias(hp->beta2, t);
  c.omb1 = 1.0 - c.b1;
  c.omb2 = 1.0 - c.b2;
  c.floor_ = hp->eps * hp->eps;
  c.eps = hp->eps;
  c.alpha = hp->alpha;
  c.wd = hp->weight_decay;
  c.update_clip = hp->clipping == SB_CLIP_UPDATE;
  if (ex && ex->loss_scale != 1.0) {
    int e2 = 0;
    const double m = std::frexp(ex->loss_scale, &e2);
    const bool pow2 = m == 0.5 && e2 - 1 >= -126 && e2 - 1 <= 126;  // 1/scale exact in fp32
    c.scale_mode = pow2 ? 1 : 2;
    c.inv_scale_f = pow2 ? static_cast<float>(1.0 / ex->loss_scale) : 0.0f;
    c.scale = ex->loss_scale;
  }

  int64_t total_blocks = 0;
  const std::vector<Group> groups = make_groups(tensors, ntensors, &total_blocks, ex);
  double* partials = static_cast<double*>(workspace);
  double* clip = partials + total_blocks;
  double* eta_buf = clip + 1;
  double* tensor_ss = eta_buf + kMaxGroup;
  unsigned int* skip_int = reinterpret_cast<unsigned int*>(tensor_ss + ntensors);
  unsigned int* amax_int = skip_int + ntensors;
  unsigned int* sync = amax_int + ntensors;

  // statistics pass: needed by the skip decision, the telemetry and the global-norm clip
  const bool stats = hp->clipping == SB_CLIP_GRAD ||
                     (ex && (ex->skipped || ex->grad_absmax || ex->loss_scale != 1.0));
  int32_t* skipped = ex && ex->skipped ? ex->skipped : reinterpret_cast<int32_t*>(skip_int);
  unsigned int* amax = ex && ex->grad_absmax ? reinterpret_cast<unsigned int*>(ex->grad_absmax) : nullptr;
  if (stats && ntensors > 0) {
    SB_CUDA_CHECK(op, cudaMemsetAsync(tensor_ss, 0, sizeof(double) * ntensors, h->stream));
    SB_CUDA_CHECK(op, cudaMemsetAsync(skipped, 0, sizeof(int32_t) * ntensors, h->stream));
    if (amax) SB_CUDA_CHECK(op, cudaMemsetAsync(amax, 0, sizeof(unsigned int) * ntensors, h->stream));
    int64_t off = 0;
    for (const Group& g : groups) {
      SB_CUDA_CHECK(op, cudaMemsetAsync(sync, 0, sizeof(unsigned int) * g.count, h->stream));
      h->launches++;
      k_gradstats<<<static_cast<unsigned>(g.total_blocks), kThreads, 0, h->stream>>>(g, c, partials, off, sync,
                                                                                       tensor_ss, skipped, amax);
      off += g.total_blocks;
    }
    h->launches++;
    k_gradstats_final<<<1, kThreads, 0, h->stream>>>(ntensors, ex ? ex->per_tensor_skip : 1, tensor_ss, skipped,
                                                     hp->clipping == SB_CLIP_GRAD, hp->max_grad_norm, clip);
    SB_LAUNCH_CHECK(op);
    c.skipped = ex ? skipped : nullptr;
  }
  // persistent task-list kernel per group; sync words (task counter + per-tensor phase-1
  // counts) zeroed once per group
  const bool extra = ex != nullptr;
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, extra ? k_adamw_persistent<true> : k_adamw_persistent<false>,
                                                kThreads, 0);
  blocks_per_sm = std::max(1, blocks_per_sm);
  for (const Group& g : groups) {
    SB_CUDA_CHECK(op, cudaMemsetAsync(sync, 0, sizeof(unsigned int) * (2 * g.count + 1), h->stream));
    const int64_t grid = std::min<int64_t>(g.total_tasks, static_cast<int64_t>(h->num_sms) * blocks_per_sm);
    h->launches++;
    const double* cp = hp->clipping == SB_CLIP_GRAD ? clip : nullptr;
    if (extra)
      k_adamw_persistent<true><<<static_cast<unsigned>(grid), kThreads, 0, h->stream>>>(g, c, cp, partials, sync, eta_buf,
                                                                                       rms_out, eta_out);
    else
      k_adamw_persistent<false><<<static_cast<unsigned>(grid), kThreads, 0, h->stream>>>(g, c, cp, partials, sync,
                                                                                        eta_buf, rms_out, eta_out);
  }
  if (rms_out || eta_out) {
    EmptyList e{};
    for (int i = 0; i < ntensors; ++i) {
      if (tensors[i].numel != 0) continue;
      e.index[e.count++] = i;
      if (e.count == 64) {
        h->launches++;
        k_empty_infos<<<1, 64, 0, h->stream>>>(e, hp->alpha, rms_out, eta_out);
        e.count = 0;
      }
    }
    if (e.count > 0) {
      h->launches++;
      k_empty_infos<<<1, 64, 0, h->stream>>>(e, hp->alpha, rms_out, eta_out);
    }
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_step(sb_handle h, const sb_adamw_tensor* tensors, int ntensors,
                                         const sb_adamw_hparams* hp, int64_t t, double* rms_out, double* eta_out,
                                         void* workspace, size_t workspace_bytes) {
  return sb_stableadamw_step_ex(h, tensors, ntensors, hp, t, nullptr, rms_out, eta_out, workspace, workspace_bytes);
}

// ------------------------------------------------------------------ ZeRO-1 ----
#define SB_TRY_O(expr)           \
  do {                           \
    const sb_status _s = (expr); \
    if (_s != SB_OK) return _s;  \
  } while (0)
__global__ void k_shard_info(const double* sum, double numel_total, double alpha, int update_clip, double* rms_out,
                             double* eta_out) {
  const double rms = __dsqrt_rn(__ddiv_rn(*sum, numel_total));
  if (rms_out) *rms_out = rms;
  if (eta_out) *eta_out = update_clip ? __ddiv_rn(alpha, rms > 1.0 ? rms : 1.0) : alpha;
}
// StableAdamW on one rank's shard of every tensor ("C5 ZeRO-1 adds reduce-scatter
// (dW) -> local StableAdamW on the shard -> all-gather(theta), plus one fp64 scalar per tensor
// (sum g^2 / max(u, eps^2)) allreduced before eta"). The RMS couples every element of a tensor
// (optimizer.cpp:148-157), so the step splits at that point: phase 1 updates v, u of the shard and
// returns the shard's sum per tensor; the caller (or sb_stableadamw_step_sharded, over the
// handle's NCCL communicator) sums them over ranks; phase 2 forms RMS over the whole tensor and
// updates theta (and, with shadow_bf16 / absmax_word, the next forward's bf16 weight rows).
// v, u are bitwise those of the unsharded step; RMS differs from it only by the order of the
// cross-rank sum (so theta is bitwise whenever eta does not depend on it, e.g. RMS <= 1 under
// update clipping). Plain steps only: no loss-scale unscaling, skipping or global-norm clip.
namespace {
sb_status shard_check(const char* op, sb_handle h, const sb_adamw_tensor* tensors, const int64_t* numel_total,
                      int ntensors, const sb_adamw_hparams* hp, int64_t t, void* workspace, size_t workspace_bytes) {
  if (!h || !hp || (ntensors > 0 && (!tensors || !numel_total)))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null argument");
  if (t < 1) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "t must be >= 1");
  if (hp->clipping == SB_CLIP_GRAD)
    return sb::fail(SB_ERR_UNSUPPORTED, op, "grad_clip needs the global norm: use the unsharded step");
  for (int i = 0; i < ntensors; ++i)
    if (tensors[i].numel < 0 || numel_total[i] < tensors[i].numel ||
        (tensors[i].numel != 0 && (!tensors[i].theta || !tensors[i].grad || !tensors[i].v || !tensors[i].u)))
      return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad tensor shard");
  size_t need = 0;
  sb_stableadamw_workspace_size(tensors, ntensors, &need);
  need += static_cast<size_t>(ntensors) * sizeof(double);
  if (!workspace || workspace_bytes < need) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  return SB_OK;
}
Coeffs shard_coeffs(const sb_adamw_hparams* hp, int64_t t) {
  Coeffs c{};
  c.b1 = debias(hp->beta1, t);
  c.b2 = hp->beta2_warmup_lambda > 0 ? beta2_warmup(t, hp->beta2_warmup_lambda) : debias(hp->beta2, t);
  c.omb1 = 1.0 - c.b1;
  c.omb2 = 1.0 - c.b2;
  c.floor_ = hp->eps * hp->eps;
  c.eps = hp->eps;
  c.alpha = hp->alpha;
  c.wd = hp->weight_decay;
  c.update_clip = hp->clipping == SB_CLIP_UPDATE;
  return c;
}
}  // namespace

extern "C" sb_status sb_stableadamw_sharded_workspace_size(const sb_adamw_tensor* tensors, int ntensors,
                                                           size_t* bytes) {
  SB_TRY_O(sb_stableadamw_workspace_size(tensors, ntensors, bytes));
  *bytes = ((*bytes + 15) & ~size_t(15)) + static_cast<size_t>(ntensors) * sizeof(double);
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_shard_phase1(sb_handle h, const sb_adamw_tensor* tensors,
                                                 const int64_t* numel_total, int ntensors,
                                                 const sb_adamw_hparams* hp, int64_t t, double* shard_sums,
                                                 void* workspace, size_t workspace_bytes) {
  const char* op = "optimizer_step_sharded";
  SB_TRY_O(shard_check(op, h, tensors, numel_total, ntensors, hp, t, workspace, workspace_bytes));
  if (ntensors > 0 && !shard_sums) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null shard_sums");
  cudaSetDevice(h->device);
  const Coeffs c = shard_coeffs(hp, t);
  int64_t total_blocks = 0;
  const std::vector<Group> groups = make_groups(tensors, ntensors, &total_blocks, nullptr, 1, numel_total);
  double* partials = static_cast<double*>(workspace);
  unsigned int* sync = reinterpret_cast<unsigned int*>(partials + total_blocks + 2 + kMaxGroup + ntensors);
  // an empty shard contributes 0 to its tensor's sum
  if (ntensors > 0) SB_CUDA_CHECK(op, cudaMemsetAsync(shard_sums, 0, sizeof(double) * ntensors, h->stream));
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_adamw_persistent<false, 1>, kThreads, 0);
  blocks_per_sm = std::max(1, blocks_per_sm);
  for (const Group& g : groups) {
    SB_CUDA_CHECK(op, cudaMemsetAsync(sync, 0, sizeof(unsigned int) * (2 * g.count + 1), h->stream));
    const int64_t grid = std::min<int64_t>(g.total_tasks, static_cast<int64_t>(h->num_sms) * blocks_per_sm);
    h->launches++;
    k_adamw_persistent<false, 1><<<static_cast<unsigned>(grid), kThreads, 0, h->stream>>>(
        g, c, nullptr, partials, sync, shard_sums, nullptr, nullptr);
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_shard_phase2(sb_handle h, const sb_adamw_tensor* tensors,
                                                 const int64_t* numel_total, int ntensors,
                                                 const sb_adamw_hparams* hp, int64_t t, const double* total_sums,
                                                 void* const* shadow_bf16, unsigned int* const* absmax_word,
                                                 double* rms_out, double* eta_out, void* workspace,
                                                 size_t workspace_bytes) {
  const char* op = "optimizer_step_sharded";
  SB_TRY_O(shard_check(op, h, tensors, numel_total, ntensors, hp, t, workspace, workspace_bytes));
  if (ntensors > 0 && !total_sums) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null total_sums");
  cudaSetDevice(h->device);
  const Coeffs c = shard_coeffs(hp, t);
  sb_adamw_extras ex{};
  ex.loss_scale = 1.0;
  ex.shadow_bf16 = shadow_bf16;
  ex.absmax_word = absmax_word;
  const bool extra = shadow_bf16 != nullptr || absmax_word != nullptr;
  int64_t total_blocks = 0;
  const std::vector<Group> groups =
      make_groups(tensors, ntensors, &total_blocks, extra ? &ex : nullptr, 2, numel_total);
  double* partials = static_cast<double*>(workspace);
  unsigned int* sync = reinterpret_cast<unsigned int*>(partials + total_blocks + 2 + kMaxGroup + ntensors);
  if (absmax_word)
    for (int i = 0; i < ntensors; ++i)
      if (absmax_word[i]) SB_CUDA_CHECK(op, cudaMemsetAsync(absmax_word[i], 0, sizeof(unsigned int), h->stream));
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, extra ? k_adamw_persistent<true, 2> : k_adamw_persistent<false, 2>,
                                                kThreads, 0);
  blocks_per_sm = std::max(1, blocks_per_sm);
  for (const Group& g : groups) {
    SB_CUDA_CHECK(op, cudaMemsetAsync(sync, 0, sizeof(unsigned int), h->stream));
    const int64_t grid = std::min<int64_t>(g.total_tasks, static_cast<int64_t>(h->num_sms) * blocks_per_sm);
    h->launches++;
    // eta_buf = the summed RMS terms, indexed by caller tensor (read only in MODE 2)
    double* sums = const_cast<double*>(total_sums);
    if (extra)
      k_adamw_persistent<true, 2><<<static_cast<unsigned>(grid), kThreads, 0, h->stream>>>(g, c, nullptr, partials, sync,
                                                                                          sums, rms_out, eta_out);
    else
      k_adamw_persistent<false, 2><<<static_cast<unsigned>(grid), kThreads, 0, h->stream>>>(g, c, nullptr, partials, sync,
                                                                                           sums, rms_out, eta_out);
  }
  // a rank whose shard of a tensor is empty still reports the tensor's rms / eta
  if (rms_out || eta_out) {
    for (int i = 0; i < ntensors; ++i) {
      if (tensors[i].numel != 0) continue;
      h->launches++;
      k_shard_info<<<1, 1, 0, h->stream>>>(total_sums + i, static_cast<double>(numel_total[i]), c.alpha,
                                           c.update_clip, rms_out ? rms_out + i : nullptr, eta_out ? eta_out + i : nullptr);
    }
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_step_sharded(sb_handle h, const sb_adamw_tensor* tensors,
                                                 const int64_t* numel_total, int ntensors,
                                                 const sb_adamw_hparams* hp, int64_t t,
                                                 void* const* shadow_bf16, unsigned int* const* absmax_word,
                                                 double* rms_out, double* eta_out, void* workspace,
                                                 size_t workspace_bytes) {
  const char* op = "optimizer_step_sharded";
  SB_TRY_O(shard_check(op, h, tensors, numel_total, ntensors, hp, t, workspace, workspace_bytes));
  size_t base = 0, need = 0;
  sb_stableadamw_workspace_size(tensors, ntensors, &base);
  sb_stableadamw_sharded_workspace_size(tensors, ntensors, &need);
  if (workspace_bytes < need) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  double* sums = reinterpret_cast<double*>(static_cast<uint8_t*>(workspace) + ((base + 15) & ~size_t(15)));
  SB_TRY_O(sb_stableadamw_shard_phase1(h, tensors, numel_total, ntensors, hp, t, sums, workspace, base + ntensors * 8));
  int rank = 0, world = 1;
  sb_dp_rank(h, &rank, &world);
  if (world > 1 && ntensors > 0) SB_TRY_O(sb_dp_allreduce_sum_f64(h, sums, ntensors));
  SB_TRY_O(sb_stableadamw_shard_phase2(h, tensors, numel_total, ntensors, hp, t, sums, shadow_bf16, absmax_word,
                                       rms_out, eta_out, workspace, base + ntensors * 8));
  // each rank's absmax words cover its rows only: the next forward's tensor-wise scale is their max
  if (world > 1 && absmax_word) SB_TRY_O(sb_dp_allreduce_max_words(h, absmax_word, ntensors));
  return SB_OK;
}
