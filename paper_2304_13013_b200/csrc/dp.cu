// dp.cu — data parallelism over the token dimension, in the C-ABI.
//
// The reference is single-process; a data-parallel SwitchBack step shards the T token rows over
// ranks (one process per GPU). Row-wise quantization and the forward / input-gradient GEMMs are
// row-independent and W (and its tensor-wise scale) is replicated, so each rank's Y / dX rows are
// bit-identical to the single-GPU result; the exchange steps are:
//   * dW = sum_r G_r^T X_r — a sum all-reduce, issued on the handle's communication stream as
//     each layer's dW GEMM finishes, so layer L's transfer overlaps layer L-1's backward;
//   * AllQuant's token-dimension quantization (linear.cpp:239-241: rows of G^T and X^T span all
//     T tokens) — a max all-reduce of the per-feature absmax words before quantizing;
//   * a ZeRO-style sharded optimizer's per-tensor sums of g^2 / max(u, eps^2) — a sum all-reduce
//     of n doubles before eta.
// NCCL is opened at run time (dlopen "libnccl.so.2": the copy the host process already loaded,
// e.g. torch's, else the system one), so the library has no link-time NCCL dependency and a
// build without NCCL still serves every single-GPU entry. Communicator setup follows NCCL's
// own: rank 0 calls sb_dp_unique_id and ships the 128 bytes to every rank out of band (MPI,
// torch.distributed, a file); each rank calls sb_dp_init(handle, id, rank, world).
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>
#include <string>

#include "sb_internal.h"

namespace {

// The slice of nccl.h this file needs (ABI-stable across NCCL 2.x).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
enum { ncclSum = 0, ncclMax = 2 };
enum { ncclUint8 = 1, ncclUint32 = 3, ncclInt64 = 4, ncclFloat32 = 7, ncclFloat64 = 8 };

struct Nccl {
  void* lib = nullptr;
  int (*getUniqueId)(ncclUniqueId*) = nullptr;
  int (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  int (*commDestroy)(ncclComm_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*reduceScatter)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  const char* (*errorString)(int) = nullptr;
  int (*getVersion)(int*) = nullptr;
  bool ok = false;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      n.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (n.lib) break;
    }
    if (!n.lib) return;
    n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(n.lib, "ncclGetUniqueId"));
    n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(n.lib, "ncclCommInitRank"));
    n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(n.lib, "ncclCommDestroy"));
    n.allReduce = reinterpret_cast<decltype(n.allReduce)>(dlsym(n.lib, "ncclAllReduce"));
    n.reduceScatter = reinterpret_cast<decltype(n.reduceScatter)>(dlsym(n.lib, "ncclReduceScatter"));
    n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(n.lib, "ncclAllGather"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(dlsym(n.lib, "ncclBroadcast"));
    n.groupStart = reinterpret_cast<decltype(n.groupStart)>(dlsym(n.lib, "ncclGroupStart"));
    n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(dlsym(n.lib, "ncclGroupEnd"));
    n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(n.lib, "ncclGetErrorString"));
    n.getVersion = reinterpret_cast<decltype(n.getVersion)>(dlsym(n.lib, "ncclGetVersion"));
    n.ok = n.getUniqueId && n.commInitRank && n.commDestroy && n.allReduce && n.reduceScatter && n.allGather &&
           n.broadcast &&
           n.groupStart && n.groupEnd && n.errorString;
  });
  return n;
}

sb_status nccl_fail(const char* op, int r) {
  std::string msg = std::string("NCCL error: ") + (nccl().errorString ? nccl().errorString(r) : "?");
  return sb::fail(SB_ERR_CUDA, op, msg.c_str());
}

#define SB_NCCL(op, expr)                     \
  do {                                        \
    const int _r = (expr);                    \
    if (_r != ncclSuccess) return nccl_fail(op, _r); \
  } while (0)

#define SB_TRY_S(expr)                 \
  do {                                 \
    const sb_status _s = (expr);       \
    if (_s != SB_OK) return _s;        \
  } while (0)

sb_status need_comm(sb_handle h, const char* op) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null handle");
  if (!h->dp_comm) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "no communicator: call sb_dp_init first");
  cudaSetDevice(h->device);
  return SB_OK;
}

__global__ void k_widen_i32(const int32_t* __restrict__ a, int64_t* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    b[i] = a[i];
}
// linear.cpp:49 over int64 accumulators: float(double(acc) * s_row * s_col / 16129.0)
__global__ void k_dequant_i64(const int64_t* __restrict__ acc, const float* __restrict__ srow,
                              const float* __restrict__ scol, int64_t rows, int64_t cols, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * cols;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    y[i] = __double2float_rn(__ddiv_rn(
        __dmul_rn(__dmul_rn(static_cast<double>(acc[i]), static_cast<double>(srow[r])), static_cast<double>(scol[c])),
        16129.0));
  }
}

}  // namespace

namespace sb {

const sb_symbuf* find_symbuf(sb_handle h, const void* p, size_t bytes) {
  const auto* q = static_cast<const uint8_t*>(p);
  for (const sb_symbuf& s : h->sym) {
    const auto* b = static_cast<const uint8_t*>(s.local);
    if (q >= b && q + bytes <= b + s.bytes) return &s;
  }
  return nullptr;
}

void dp_owned_rows(int64_t rows, int rank, int world, int64_t* r0, int64_t* r1) {
  const int64_t nb = (rows + 31) / 32;
  auto first_block = [&](int64_t r) { return (r * nb + world - 1) / world; };  // ceil(r nb / world)
  *r0 = std::min<int64_t>(rows, 32 * first_block(rank));
  *r1 = std::min<int64_t>(rows, 32 * first_block(rank + 1));
}

sb_status dp_allreduce_sum_f32(sb_handle h, float* buf, int64_t n, cudaStream_t stream) {
  const char* op = "dp_allreduce";
  if (!h->dp_comm || h->dp_world <= 1 || n <= 0) return SB_OK;
  SB_NCCL(op, nccl().allReduce(buf, buf, static_cast<size_t>(n), ncclFloat32, ncclSum,
                               static_cast<ncclComm_t>(h->dp_comm), stream));
  return SB_OK;
}

void dp_free_symmetric(sb_handle h) {
  for (sb_symbuf& s : h->sym) {
    for (int r = 0; r < s.world; ++r)
      if (s.opened && r != s.rank && s.peer[r]) cudaIpcCloseMemHandle(s.peer[r]);
    cudaFree(s.local);
  }
  h->sym.clear();
}

bool dp_active(sb_handle h) {
  static int force = -1;
  if (force < 0) force = getenv("SB_DP_FORCE") ? atoi(getenv("SB_DP_FORCE")) : 0;
  return h->dp_comm != nullptr && (h->dp_world > 1 || force != 0);
}

sb_status dp_allquant_dw(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t n, int64_t m,
                         int8_t* gt_q, float* gt_state, int8_t* xt_q, float* xt_state, unsigned int* words,
                         int64_t* raw64, float* dw) {
  const char* op = "linear_backward";
  auto comm = static_cast<ncclComm_t>(h->dp_comm);
  // G^T rows = G's columns (m features over all tokens), X^T rows = X's columns (n features)
  SB_CUDA_CHECK(op, sb::launch_absmax_columns(h, g, dt, b, m, m, words));
  SB_NCCL(op, nccl().allReduce(words, words, static_cast<size_t>(m), ncclUint32, ncclMax, comm, h->stream));
  SB_CUDA_CHECK(op, sb::launch_quantize_from_words(h, g, dt, b, m, m, words, 1, nullptr, 0, gt_q, b, gt_state));
  SB_CUDA_CHECK(op, sb::launch_absmax_columns(h, x, dt, b, n, n, words));
  SB_NCCL(op, nccl().allReduce(words, words, static_cast<size_t>(n), ncclUint32, ncclMax, comm, h->stream));
  SB_CUDA_CHECK(op, sb::launch_quantize_from_words(h, x, dt, b, n, n, words, 1, nullptr, 0, xt_q, b, xt_state));
  // this rank's integer product over its b tokens (|acc| <= 127^2 b: int32 up to b = 133144)
  if (b > 133144) return sb::fail(SB_ERR_UNSUPPORTED, op, "AllQuant under data parallelism: > 133144 tokens per rank");
  const sb_status st = sb::gemm_i8(h, gt_q, nullptr, xt_q, nullptr, SB_SCALE_NONE, m, n, b, dw, SB_I32, 0);
  if (st != SB_OK) return st;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((m * n + 255) / 256, 4 * 148));
  h->launches += 2;
  k_widen_i32<<<grid, 256, 0, h->stream>>>(reinterpret_cast<const int32_t*>(dw), raw64, m * n);
  SB_NCCL(op, nccl().allReduce(raw64, raw64, static_cast<size_t>(m * n), ncclInt64, ncclSum, comm, h->stream));
  k_dequant_i64<<<grid, 256, 0, h->stream>>>(raw64, gt_state, xt_state, m, n, dw);
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

}  // namespace sb

extern "C" {

sb_status sb_dp_available(int* version) {
  Nccl& n = nccl();
  if (!n.ok) return sb::fail(SB_ERR_UNSUPPORTED, "sb_dp_available", "libnccl.so.2 not found");
  if (version) {
    *version = 0;
    if (n.getVersion) n.getVersion(version);
  }
  return SB_OK;
}

sb_status sb_dp_unique_id(uint8_t* id_out) {
  const char* op = "sb_dp_unique_id";
  if (!id_out) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null id");
  SB_TRY_S(sb_dp_available(nullptr));
  ncclUniqueId id;
  SB_NCCL(op, nccl().getUniqueId(&id));
  std::memcpy(id_out, id.internal, sizeof(id.internal));
  return SB_OK;
}

sb_status sb_dp_init(sb_handle h, const uint8_t* id, int rank, int world) {
  const char* op = "sb_dp_init";
  if (!h || !id || world < 1 || rank < 0 || rank >= world) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_TRY_S(sb_dp_available(nullptr));
  if (h->dp_comm) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "communicator already initialised");
  cudaSetDevice(h->device);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  ncclComm_t comm = nullptr;
  SB_NCCL(op, nccl().commInitRank(&comm, world, uid, rank));
  h->dp_comm = comm;
  h->dp_rank = rank;
  h->dp_world = world;
  SB_CUDA_CHECK(op, cudaStreamCreateWithFlags(&h->dp_stream, cudaStreamNonBlocking));
  SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&h->dp_ready, cudaEventDisableTiming));
  SB_CUDA_CHECK(op, cudaEventCreateWithFlags(&h->dp_done, cudaEventDisableTiming));
  if (!h->dp_token) SB_CUDA_CHECK(op, cudaMalloc(&h->dp_token, sizeof(float)));
  if (getenv("SB_DEBUG") || getenv("SB_DP_LOG")) {
    int v = 0;
    if (nccl().getVersion) nccl().getVersion(&v);
    fprintf(stderr, "[sb] dp: rank %d of %d on device %d, NCCL %d\n", rank, world, h->device, v);
  }
  return SB_OK;
}

sb_status sb_dp_rank(sb_handle h, int* rank, int* world) {
  if (!h || !rank || !world) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_dp_rank", "bad argument");
  *rank = h->dp_comm ? h->dp_rank : 0;
  *world = h->dp_comm ? h->dp_world : 1;
  return SB_OK;
}

// Sum all-reduce of fp32 gradients, in place, on the communication stream after everything
// enqueued so far on the handle's stream; returns at once. ncclGroup fuses the buffers into one
// launch. A plain sum, like the reference's dW over the batch rows (linear.cpp:245).
sb_status sb_dp_allreduce_grads_async(sb_handle h, float* const* bufs, const int64_t* numel, int n) {
  const char* op = "sb_dp_allreduce_grads";
  SB_TRY_S(need_comm(h, op));
  if (n < 0 || (n > 0 && (!bufs || !numel))) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_CUDA_CHECK(op, cudaEventRecord(h->dp_ready, h->stream));
  SB_CUDA_CHECK(op, cudaStreamWaitEvent(h->dp_stream, h->dp_ready, 0));
  SB_NCCL(op, nccl().groupStart());
  for (int i = 0; i < n; ++i)
    if (numel[i] > 0)
      SB_NCCL(op, nccl().allReduce(bufs[i], bufs[i], static_cast<size_t>(numel[i]), ncclFloat32, ncclSum,
                                   static_cast<ncclComm_t>(h->dp_comm), h->dp_stream));
  SB_NCCL(op, nccl().groupEnd());
  SB_CUDA_CHECK(op, cudaEventRecord(h->dp_done, h->dp_stream));
  h->dp_pending = true;
  return SB_OK;
}

// Make the handle's stream wait for every all-reduce issued so far (no host block).
sb_status sb_dp_wait(sb_handle h) {
  const char* op = "sb_dp_wait";
  SB_TRY_S(need_comm(h, op));
  if (h->dp_pending) SB_CUDA_CHECK(op, cudaStreamWaitEvent(h->stream, h->dp_done, 0));
  h->dp_pending = false;
  return SB_OK;
}

// Synchronous (stream-ordered on the handle's stream) all-reduces of small vectors:
// max of uint32 words (absmax bit patterns: AllQuant across ranks) and sum of doubles.
sb_status sb_dp_allreduce_max_u32(sb_handle h, unsigned int* words, int64_t n) {
  const char* op = "sb_dp_allreduce_max";
  SB_TRY_S(need_comm(h, op));
  if (n <= 0) return SB_OK;
  SB_NCCL(op, nccl().allReduce(words, words, static_cast<size_t>(n), ncclUint32, ncclMax,
                               static_cast<ncclComm_t>(h->dp_comm), h->stream));
  return SB_OK;
}

// Max all-reduce of n separate device words in one NCCL group (the ZeRO-1 step's per-tensor bf16
// shadow absmax words: each rank saw only its rows).
sb_status sb_dp_allreduce_max_words(sb_handle h, unsigned int* const* words, int n) {
  const char* op = "sb_dp_allreduce_max";
  SB_TRY_S(need_comm(h, op));
  if (n < 0 || (n > 0 && !words)) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_NCCL(op, nccl().groupStart());
  for (int i = 0; i < n; ++i)
    if (words[i])
      SB_NCCL(op, nccl().allReduce(words[i], words[i], 1, ncclUint32, ncclMax, static_cast<ncclComm_t>(h->dp_comm),
                                   h->stream));
  SB_NCCL(op, nccl().groupEnd());
  return SB_OK;
}

sb_status sb_dp_allreduce_sum_f64(sb_handle h, double* vals, int64_t n) {
  const char* op = "sb_dp_allreduce_sum";
  SB_TRY_S(need_comm(h, op));
  if (n <= 0) return SB_OK;
  SB_NCCL(op, nccl().allReduce(vals, vals, static_cast<size_t>(n), ncclFloat64, ncclSum,
                               static_cast<ncclComm_t>(h->dp_comm), h->stream));
  return SB_OK;
}

sb_status sb_dp_destroy(sb_handle h) {
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_dp_destroy", "null handle");
  if (!h->dp_comm) return SB_OK;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->dp_stream);
  nccl().commDestroy(static_cast<ncclComm_t>(h->dp_comm));
  h->dp_comm = nullptr;
  cudaStreamDestroy(h->dp_stream);
  cudaEventDestroy(h->dp_ready);
  cudaEventDestroy(h->dp_done);
  h->dp_stream = nullptr;
  if (h->dp_token) cudaFree(h->dp_token);
  h->dp_token = nullptr;
  return SB_OK;
}

// ------------------------------------------------ fused dW reduce-scatter ---
// Symmetric buffers: cudaMalloc'ed on every rank, exported with cudaIpcGetMemHandle, and every
// peer's copy opened in this process, so the dW kernel's epilogue can TMA reduce-add into the
// owner's copy over NVLink (P2P). The handles travel out of band (sb_dp_symmetric_open) or over
// the handle's NCCL communicator (sb_dp_symmetric_exchange).
sb_status sb_dp_symmetric_alloc(sb_handle h, size_t bytes, void** ptr, uint8_t* ipc_handle) {
  const char* op = "sb_dp_symmetric_alloc";
  if (!h || !ptr || !ipc_handle || bytes == 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  cudaSetDevice(h->device);
  sb_symbuf s;
  s.bytes = (bytes + 255) & ~size_t(255);
  SB_CUDA_CHECK(op, cudaMalloc(&s.local, s.bytes));
  cudaIpcMemHandle_t ih;
  const cudaError_t e = cudaIpcGetMemHandle(&ih, s.local);
  if (e != cudaSuccess) {
    cudaFree(s.local);
    return sb::cuda_fail(op, e);
  }
  std::memcpy(ipc_handle, &ih, sizeof(ih));
  h->sym.push_back(s);
  *ptr = s.local;
  return SB_OK;
}

sb_status sb_dp_symmetric_open(sb_handle h, void* ptr, int rank, int world, const uint8_t* ipc_handles) {
  const char* op = "sb_dp_symmetric_open";
  if (!h || !ptr || !ipc_handles || world < 1 || world > 8 || rank < 0 || rank >= world)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument (1 <= world <= 8)");
  sb_symbuf* s = const_cast<sb_symbuf*>(sb::find_symbuf(h, ptr, 1));
  if (!s || s->local != ptr) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "not a symmetric buffer of this handle");
  if (s->opened) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "already opened");
  cudaSetDevice(h->device);
  s->rank = rank;
  s->world = world;
  for (int r = 0; r < world; ++r) {
    if (r == rank) {
      s->peer[r] = s->local;
      continue;
    }
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, ipc_handles + 64 * r, sizeof(ih));
    const cudaError_t e = cudaIpcOpenMemHandle(&s->peer[r], ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int q = 0; q < r; ++q)
        if (q != rank && s->peer[q]) cudaIpcCloseMemHandle(s->peer[q]);
      std::memset(s->peer, 0, sizeof(s->peer));
      return sb::cuda_fail(op, e);
    }
  }
  s->opened = true;
  return SB_OK;
}

sb_status sb_dp_symmetric_exchange(sb_handle h, void* ptr, const uint8_t* ipc_handle) {
  const char* op = "sb_dp_symmetric_exchange";
  SB_TRY_S(need_comm(h, op));
  if (!ptr || !ipc_handle) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  if (h->dp_world > 8) return sb::fail(SB_ERR_UNSUPPORTED, op, "at most 8 ranks");
  uint8_t* d = nullptr;
  SB_CUDA_CHECK(op, cudaMalloc(&d, 64 * static_cast<size_t>(h->dp_world)));
  std::vector<uint8_t> all(64 * static_cast<size_t>(h->dp_world));
  cudaError_t e = cudaMemcpyAsync(d + 64 * h->dp_rank, ipc_handle, 64, cudaMemcpyHostToDevice, h->stream);
  int r = ncclSuccess;
  if (e == cudaSuccess)
    r = nccl().allGather(d + 64 * h->dp_rank, d, 64, ncclUint8, static_cast<ncclComm_t>(h->dp_comm), h->stream);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaMemcpyAsync(all.data(), d, all.size(), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(h->stream);
  cudaFree(d);
  if (r != ncclSuccess) return nccl_fail(op, r);
  if (e != cudaSuccess) return sb::cuda_fail(op, e);
  return sb_dp_symmetric_open(h, ptr, h->dp_rank, h->dp_world, all.data());
}

sb_status sb_dp_symmetric_free(sb_handle h, void* ptr) {
  const char* op = "sb_dp_symmetric_free";
  if (!h) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "null handle");
  for (size_t i = 0; i < h->sym.size(); ++i) {
    sb_symbuf& s = h->sym[i];
    if (s.local != ptr) continue;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (int r = 0; r < s.world; ++r)
      if (s.opened && r != s.rank && s.peer[r]) cudaIpcCloseMemHandle(s.peer[r]);
    cudaFree(s.local);
    h->sym.erase(h->sym.begin() + static_cast<std::ptrdiff_t>(i));
    return SB_OK;
  }
  return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "not a symmetric buffer of this handle");
}

sb_status sb_dp_owned_rows(int64_t rows, int rank, int world, int64_t* r0, int64_t* r1) {
  if (rows < 0 || world < 1 || rank < 0 || rank >= world || !r0 || !r1)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, "sb_dp_owned_rows", "bad argument");
  sb::dp_owned_rows(rows, rank, world, r0, r1);
  return SB_OK;
}

sb_status sb_wgrad_reduce_scatter(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                  int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state) {
  const char* op = "wgrad_reduce_scatter";
  if (!h || !g || !x || !dw || b <= 0 || m <= 0 || n <= 0 || (g_q && (!g_state || ldq < m)))
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  const sb_symbuf* s = sb::find_symbuf(h, dw, static_cast<size_t>(m * n) * sizeof(float));
  if (!s) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "dw is not inside a symmetric buffer (sb_dp_symmetric_alloc)");
  cudaSetDevice(h->device);
  const sb::RowQuant rq{g_q, ldq, g_state};
  return sb::wgrad_reduce_scatter(h, g, x, dt, b, m, n, dw, *s, g_q ? &rq : nullptr);
}

// Stream-ordered barrier: a one-element all-reduce on the handle's stream. When it completes on
// a rank, every rank has reached it (and finished the work it enqueued before it).
sb_status sb_dp_barrier(sb_handle h) {
  const char* op = "sb_dp_barrier";
  SB_TRY_S(need_comm(h, op));
  SB_NCCL(op, nccl().allReduce(h->dp_token, h->dp_token, 1, ncclFloat32, ncclSum, static_cast<ncclComm_t>(h->dp_comm),
                               h->stream));
  return SB_OK;
}

// After the reduce-scatter each rank's copy holds the complete sum in the rows it owns; every
// owner broadcasts its rows into the same rows of the other ranks' copies (one NCCL group).
sb_status sb_dp_allgather_rows(sb_handle h, float* dw, int64_t m, int64_t n) {
  const char* op = "sb_dp_allgather_rows";
  SB_TRY_S(need_comm(h, op));
  if (!dw || m <= 0 || n <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  SB_NCCL(op, nccl().groupStart());
  for (int r = 0; r < h->dp_world; ++r) {
    int64_t r0 = 0, r1 = 0;
    sb::dp_owned_rows(m, r, h->dp_world, &r0, &r1);
    if (r1 > r0)
      SB_NCCL(op, nccl().broadcast(dw + r0 * n, dw + r0 * n, static_cast<size_t>((r1 - r0) * n), ncclFloat32, r,
                                   static_cast<ncclComm_t>(h->dp_comm), h->stream));
  }
  SB_NCCL(op, nccl().groupEnd());
  return SB_OK;
}

// The whole fused exchange for one weight gradient, stream-ordered on the handle's stream:
// zero this rank's copy, barrier (every copy zeroed before any rank adds), the dW GEMM with its
// reduce-scatter epilogue, barrier (every rank's adds landed), all-gather of the owned rows.
// Afterwards dw holds sum_r G_r^T X_r on every rank. Without a communicator (one rank) it is
// the GEMM into the zeroed local buffer.
sb_status sb_dp_wgrad_allreduce_fused(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                      int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state) {
  const char* op = "wgrad_allreduce_fused";
  if (!h || !dw || m <= 0 || n <= 0) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "bad argument");
  const bool multi = h->dp_comm != nullptr && h->dp_world > 1;
  const sb_symbuf* sym = sb::find_symbuf(h, dw, static_cast<size_t>(m * n) * sizeof(float));
  if (sym && sym->world > 1 && !multi)
    return sb::fail(SB_ERR_INVALID_ARGUMENT, op,
                    "a multi-rank symmetric buffer needs the handle's communicator for the barriers and all-gather "
                    "(or call sb_wgrad_reduce_scatter with your own barriers)");
  if (!sym) return sb::fail(SB_ERR_INVALID_ARGUMENT, op, "dw is not inside a symmetric buffer (sb_dp_symmetric_alloc)");
  // shapes the one-wave dW kernel does not serve (e.g. a 1280 x 1280 out-projection): the local
  // GEMM (with G's quantize) and a NCCL sum all-reduce, same result contract
  const sb::RowQuant rq{g_q, ldq, g_state};
  if (!sb::dw_wide_serves(h, m, n, b) || dt != SB_BF16) {
    cudaSetDevice(h->device);
    SB_TRY_S(sb::wgrad(h, g, x, dt, b, m, n, dw, 0, 0, g_q ? &rq : nullptr));
    if (multi)
      SB_NCCL(op, nccl().allReduce(dw, dw, static_cast<size_t>(m * n), ncclFloat32, ncclSum,
                                   static_cast<ncclComm_t>(h->dp_comm), h->stream));
    return SB_OK;
  }
  SB_CUDA_CHECK(op, cudaMemsetAsync(dw, 0, static_cast<size_t>(m * n) * sizeof(float), h->stream));
  if (multi) SB_TRY_S(sb_dp_barrier(h));
  SB_TRY_S(sb_wgrad_reduce_scatter(h, g, x, dt, b, m, n, dw, g_q, ldq, g_state));
  if (multi) {
    SB_TRY_S(sb_dp_barrier(h));
    SB_TRY_S(sb_dp_allgather_rows(h, dw, m, n));
  }
  return SB_OK;
}

}  // extern "C"
