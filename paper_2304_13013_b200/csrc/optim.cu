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

#include "sb_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 16;
constexpr int kChunk = kThreads * kPerThread;  // elements per block
constexpr int kMaxGroup = 96;                  // tensors per launch (kernel-parameter budget)
constexpr size_t kGroupL2Bytes = 48ull << 20;  // v,u bytes per group kept L2-resident

struct TensorDesc {
  float* theta;
  const float* grad;
  float* v;
  float* u;
  int64_t numel;
  int64_t block0;  // first block of this tensor in the group launch
  int64_t nblocks;
  int32_t index;  // position in the caller's tensor list (rms/eta outputs)
};

struct Group {
  TensorDesc t[kMaxGroup];
  int count;
  int64_t total_blocks;
};

struct Coeffs {
  double b1, omb1, b2, omb2;  // debiased decay rates and their complements (host-computed)
  double floor_;              // eps^2
  double eps, alpha, wd;
  int32_t update_clip;
};

__device__ __forceinline__ int find_tensor(const Group& g, int64_t blk) {
  int lo = 0, hi = g.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (g.t[mid].block0 <= blk) lo = mid;
    else hi = mid - 1;
  }
  return lo;
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
  return s;
}

__global__ void __launch_bounds__(kThreads) k_adamw_phase1(const __grid_constant__ Group grp, Coeffs c,
                                                           const double* __restrict__ clip_ptr,
                                                           double* __restrict__ partials) {
  __shared__ double red[kThreads / 32];
  const int64_t blk = blockIdx.x;
  const TensorDesc& d = grp.t[find_tensor(grp, blk)];
  const int64_t base = (blk - d.block0) * kChunk;
  const double clip = clip_ptr ? *clip_ptr : 1.0;
  double acc = 0.0;
#pragma unroll 4
  for (int e = 0; e < kPerThread; ++e) {
    const int64_t i = base + e * kThreads + threadIdx.x;
    if (i < d.numel) {
      const double g = __dmul_rn(static_cast<double>(d.grad[i]), clip);
      const float vn = __double2float_rn(__dadd_rn(__dmul_rn(c.b1, static_cast<double>(d.v[i])), __dmul_rn(c.omb1, g)));
      const float un =
          __double2float_rn(__dadd_rn(__dmul_rn(c.b2, static_cast<double>(d.u[i])), __dmul_rn(__dmul_rn(c.omb2, g), g)));
      d.v[i] = vn;
      d.u[i] = un;
      const double ud = static_cast<double>(un);
      acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(g, g), ud > c.floor_ ? ud : c.floor_));
    }
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partials[blk] = s;
}

__global__ void __launch_bounds__(kThreads) k_adamw_phase2(const __grid_constant__ Group grp, Coeffs c,
                                                           const double* __restrict__ partials, double* rms_out,
                                                           double* eta_out) {
  __shared__ double red[kThreads / 32];
  __shared__ double eta_s;
  const int64_t blk = blockIdx.x;
  const TensorDesc& d = grp.t[find_tensor(grp, blk)];
  // every block of the tensor reduces the same partials in the same order -> same eta
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < d.nblocks; j += kThreads) s = __dadd_rn(s, partials[d.block0 + j]);
  // fixed-order combine of the per-thread strided sums
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0) {
    const double rms = __dsqrt_rn(__ddiv_rn(tot, static_cast<double>(d.numel)));
    const double eta = c.update_clip ? __ddiv_rn(c.alpha, rms > 1.0 ? rms : 1.0) : c.alpha;
    eta_s = eta;
    if (blk == d.block0) {
      if (rms_out) rms_out[d.index] = rms;
      if (eta_out) eta_out[d.index] = eta;
    }
  }
  __syncthreads();
  const double eta = eta_s;
  const double eta_wd = __dmul_rn(eta, c.wd);
  const int64_t base = (blk - d.block0) * kChunk;
#pragma unroll 4
  for (int e = 0; e < kPerThread; ++e) {
    const int64_t i = base + e * kThreads + threadIdx.x;
    if (i < d.numel) {
      const double th = static_cast<double>(d.theta[i]);
      const double upd = __ddiv_rn(static_cast<double>(d.v[i]), __dadd_rn(__dsqrt_rn(static_cast<double>(d.u[i])), c.eps));
      d.theta[i] = __double2float_rn(__dsub_rn(__dsub_rn(th, __dmul_rn(eta_wd, th)), __dmul_rn(eta, upd)));
    }
  }
}

// kGradClip (optimizer.cpp:121-131): global sum of squares -> clip factor on device.
__global__ void __launch_bounds__(kThreads) k_sumsq(const __grid_constant__ Group grp, double* __restrict__ partials,
                                                    int64_t offset) {
  __shared__ double red[kThreads / 32];
  const int64_t blk = blockIdx.x;
  const TensorDesc& d = grp.t[find_tensor(grp, blk)];
  const int64_t base = (blk - d.block0) * kChunk;
  double acc = 0.0;
  for (int e = 0; e < kPerThread; ++e) {
    const int64_t i = base + e * kThreads + threadIdx.x;
    if (i < d.numel) {
      const double g = static_cast<double>(d.grad[i]);
      acc = __dadd_rn(acc, __dmul_rn(g, g));
    }
  }
  const double s = block_sum(acc, red);
  if (threadIdx.x == 0) partials[offset + blk] = s;
}

__global__ void k_clip_factor(const double* __restrict__ partials, int64_t n, double max_norm, double* clip) {
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += kThreads) s = __dadd_rn(s, partials[j]);
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0) {
    const double norm = __dsqrt_rn(tot);
    *clip = norm > max_norm ? __ddiv_rn(max_norm, norm) : 1.0;
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

std::vector<Group> make_groups(const sb_adamw_tensor* ts, int n, int64_t* total_blocks) {
  std::vector<Group> groups;
  Group cur{};
  size_t cur_bytes = 0;
  int64_t blocks_all = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t nb = (ts[i].numel + kChunk - 1) / kChunk;
    const size_t bytes = static_cast<size_t>(ts[i].numel) * 8;
    if (cur.count > 0 && (cur.count == kMaxGroup || cur_bytes + bytes > kGroupL2Bytes)) {
      groups.push_back(cur);
      cur = Group{};
      cur_bytes = 0;
    }
    if (nb == 0) continue;
    TensorDesc& d = cur.t[cur.count++];
    d.theta = ts[i].theta;
    d.grad = ts[i].grad;
    d.v = ts[i].v;
    d.u = ts[i].u;
    d.numel = ts[i].numel;
    d.block0 = cur.total_blocks;
    d.nblocks = nb;
    d.index = i;
    cur.total_blocks += nb;
    cur_bytes += bytes;
    blocks_all += nb;
  }
  if (cur.count > 0) groups.push_back(cur);
  *total_blocks = blocks_all;
  return groups;
}

}  // namespace

extern "C" sb_status sb_stableadamw_workspace_size(const sb_adamw_tensor* tensors, int ntensors, size_t* bytes) {
  if (!bytes || (ntensors > 0 && !tensors)) return sb::fail(SB_ERR_INVALID_ARGUMENT, "optimizer_step", "null argument");
  int64_t total = 0;
  for (int i = 0; i < ntensors; ++i) total += (tensors[i].numel + kChunk - 1) / kChunk;
  *bytes = static_cast<size_t>(total + 16) * sizeof(double);
  return SB_OK;
}

extern "C" sb_status sb_stableadamw_step(sb_handle h, const sb_adamw_tensor* tensors, int ntensors,
                                         const sb_adamw_hparams* hp, int64_t t, double* rms_out, double* eta_out,
                                         void* workspace, size_t workspace_bytes) {
  const char* op = "optimizer_step";
  if (!h || !hp) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null argument");
  if (t < 1) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "t must be >= 1");  // optimizer.cpp:104
  for (int i = 0; i < ntensors; ++i)
    if (!tensors[i].theta || !tensors[i].grad || !tensors[i].v || !tensors[i].u || tensors[i].numel < 0)
      return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null tensor reference");  // :107-108
  if (hp->clipping == SB_CLIP_GRAD && !(hp->max_grad_norm > 0))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "max_grad_norm must be > 0");
  size_t need = 0;
  sb_stableadamw_workspace_size(tensors, ntensors, &need);
  if (!workspace || workspace_bytes < need) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "workspace too small");
  cudaSetDevice(h->device);

  Coeffs c;
  c.b1 = debias(hp->beta1, t);
  c.b2 = hp->beta2_warmup_lambda > 0 ? beta2_warmup(t, hp->beta2_warmup_lambda) : debias(hp->beta2, t);
  c.omb1 = 1.0 - c.b1;
  c.omb2 = 1.0 - c.b2;
  c.floor_ = hp->eps * hp->eps;
  c.eps = hp->eps;
  c.alpha = hp->alpha;
  c.wd = hp->weight_decay;
  c.update_clip = hp->clipping == SB_CLIP_UPDATE;

  int64_t total_blocks = 0;
  const std::vector<Group> groups = make_groups(tensors, ntensors, &total_blocks);
  double* partials = static_cast<double*>(workspace);
  double* clip = partials + total_blocks;

  if (hp->clipping == SB_CLIP_GRAD) {
    int64_t off = 0;
    for (const Group& g : groups) {
      h->launches++;
      k_sumsq<<<static_cast<unsigned>(g.total_blocks), kThreads, 0, h->stream>>>(g, partials, off);
      off += g.total_blocks;
    }
    h->launches++;
    k_clip_factor<<<1, kThreads, 0, h->stream>>>(partials, off, hp->max_grad_norm, clip);
    SB_LAUNCH_CHECK(op);
  }
  for (const Group& g : groups) {
    h->launches += 2;
    k_adamw_phase1<<<static_cast<unsigned>(g.total_blocks), kThreads, 0, h->stream>>>(
        g, c, hp->clipping == SB_CLIP_GRAD ? clip : nullptr, partials);
    k_adamw_phase2<<<static_cast<unsigned>(g.total_blocks), kThreads, 0, h->stream>>>(g, c, partials, rms_out, eta_out);
  }
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}
