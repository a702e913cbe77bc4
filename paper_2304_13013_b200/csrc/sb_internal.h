// sb_internal.h — shared host-side plumbing for the C-ABI implementation.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <vector>
#include <string>
#include <utility>

#include "../../include/switchback_b200.h"

// A symmetric buffer for the fused dW reduce-scatter: the same-size allocation on every rank,
// each rank's mapped into this process (CUDA IPC), so a kernel can reduce-add into a peer's
// copy over NVLink. peer[rank] == local.
struct sb_symbuf {
  void* local = nullptr;
  size_t bytes = 0;
  int rank = 0, world = 1;
  void* peer[8] = {};
  bool opened = false;  // peer[] filled by sb_dp_symmetric_open
};

struct sb_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  uint32_t* d_err = nullptr;       // device error latch (bit 0: non-finite input seen)
  // small per-stream scratch (tensor absmax words etc.) for the standalone ops that have no
  // caller workspace: one buffer per CUDA stream the handle has been bound to, so ops enqueued
  // eagerly on two streams never share words; allocated only outside stream capture
  std::map<cudaStream_t, std::pair<unsigned int*, size_t>> scratch;
  unsigned int* capture_scratch = nullptr;  // 1 MB from sb_create: streams first seen while capturing
  size_t capture_scratch_bytes = 0;
  uint64_t launches = 0;
  int gemm_path = 0;  // sb_gemm_path
  // host-buffer pipeline (sb_switchback_fwd_bwd_host): copy streams + events, created once
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t hp_ev[5][8] = {};  // [in, y, comp, out, x in][slot] (host pipeline, up to 8 slots)
  cudaEvent_t hp_start = nullptr;
  cudaEvent_t hp_wready = nullptr;   // MLP host pipeline: both weights uploaded
  cudaEvent_t hp_w1ready = nullptr;  // MLP host pipeline: W1 uploaded
  // two device pools used by alternate host-pipeline calls, so an async call's transfers
  // overlap the previous call's drain without aliasing its buffers
  void* dev_pool[2] = {nullptr, nullptr};
  size_t dev_pool_bytes[2] = {0, 0};
  cudaEvent_t pool_done[2] = {nullptr, nullptr};  // recorded when a call's last D2H finished
  bool pool_used[2] = {false, false};
  int pool_next = 0;
  void* gelu_lut = nullptr;  // GELU / GELU' tables for bf16 |x| < 8 (built at sb_create)
  // data parallelism (dp.cu): NCCL communicator, its stream and the fork / join events
  void* dp_comm = nullptr;
  int dp_rank = 0, dp_world = 1;
  cudaStream_t dp_stream = nullptr;
  cudaEvent_t dp_ready = nullptr, dp_done = nullptr;
  bool dp_pending = false;
  float* dp_token = nullptr;  // one device float: the payload of sb_dp_barrier's all-reduce
  std::vector<sb_symbuf> sym;  // symmetric buffers (sb_dp_symmetric_alloc)
};

namespace sb {

// SB_PDL=1 in the environment turns programmatic dependent launch on (off by default: the C2
// step measured ~1% slower with it, 23.4 vs 23.6 M tokens/s).
bool pdl_enabled();

// Launch a kernel that calls sbptx::pdl_wait() before its first global-memory access with the
// programmatic-stream-serialization attribute (ordinary stream order when PDL is off).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Thread-local "<op>: <reason>" error text (sb_last_error).
void set_error(const std::string& msg);
sb_status fail(sb_status st, const char* op, const char* reason);
sb_status cuda_fail(const char* op, cudaError_t e);

#define SB_CUDA_CHECK(op, expr)                    \
  do {                                             \
    cudaError_t _e = (expr);                       \
    if (_e != cudaSuccess) return sb::cuda_fail(op, _e); \
  } while (0)

#define SB_LAUNCH_CHECK(op)                                 \
  do {                                                      \
    cudaError_t _e = cudaGetLastError();                    \
    if (_e != cudaSuccess) return sb::cuda_fail(op, _e);    \
  } while (0)

inline size_t dt_size(sb_dtype dt) {
  switch (dt) {
    case SB_F32: return 4;
    case SB_BF16: return 2;
    case SB_I32: return 4;
    case SB_I8: return 1;
    case SB_U8: return 1;
    case SB_I64: return 8;
  }
  return 0;
}
__host__ __device__ inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

// Scratch words (device, unsigned) owned by the handle; grows on demand (not on hot path
// after the first call at a given size).
unsigned int* scratch(sb_handle h, size_t words);

// TMA tensor-map encoding through the driver entry point (no -lcuda link).
bool encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz);

// ----------------------------------------------------------- launchers ----
// quantize.cu
cudaError_t launch_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                    int8_t* q, int64_t ldq, float* state);
cudaError_t launch_absmax_tensor(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 unsigned int* word);
// Tensor-wise quantize in one launch (absmax tasks, then quantize + transpose tasks); sync = 4
// device words. Returns false (nothing launched) when x is not 16-byte vectorisable.
bool launch_quantize_tensorwise_fused(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                      int64_t ldx, int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state,
                                      unsigned int* sync, cudaError_t* err);
cudaError_t launch_absmax_columns(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                  unsigned int* words);
// Quantize with states from absmax words (tensor: one word; column: cols words);
// writes q and/or q_t; also writes the float states (sentinel applied).
cudaError_t launch_quantize_from_words(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                       int64_t ldx, const unsigned int* words, int per_column, int8_t* q, int64_t ldq,
                                       int8_t* q_t, int64_t ldqt, float* state);
cudaError_t launch_dequantize(sb_handle h, const int8_t* q, int64_t rows, int64_t cols, int64_t ldq,
                              const float* state, int axis, void* y, sb_dtype ydt, int64_t ldy);
bool launch_quantize_fp8_fast(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                              int fmt, int axis, const unsigned int* words, uint8_t* q, int64_t ldq, float* state,
                              bool row_fused, cudaError_t* err);
cudaError_t launch_quantize_fp8(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                int fmt, int axis, const unsigned int* words, uint8_t* q, int64_t ldq, float* state);
cudaError_t launch_absmax_rows(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                               unsigned int* words);
cudaError_t launch_dequantize_fp8(sb_handle h, const uint8_t* q, int64_t rows, int64_t cols, int64_t ldq, int fmt,
                                  const float* state, int axis, void* y, sb_dtype ydt, int64_t ldy);
cudaError_t launch_convert(sb_handle h, const void* x, sb_dtype xdt, void* y, sb_dtype ydt, int64_t n);
cudaError_t build_gelu_lut(sb_handle h);
int64_t ln_backward_blocks(sb_handle h);
// LayerNorm backward (bf16 dh / x / dx, fp32 mean / rstd / gamma / dgamma / dbeta) for rows of
// <= 1280 columns; part = ln_backward_blocks(h) * 2 * cols floats of scratch.
cudaError_t launch_ln_backward(sb_handle h, const void* dh, const void* x, int64_t rows, int64_t cols,
                               const float* mean, const float* rstd, const float* gamma, void* dx, float* dgamma,
                               float* dbeta, float* part);
// Fused LayerNorm (bf16 in, fp32 gamma/beta) + row-wise quantize of its bf16 output;
// cudaErrorNotSupported for rows longer than 2048 or unaligned operands.
cudaError_t launch_ln_quantize_rowwise(sb_handle h, const void* x, int64_t rows, int64_t cols, const float* gamma,
                                       const float* beta, float eps, void* out, int8_t* q, float* state, float* mean,
                                       float* rstd);
// Fused activation + row-wise quantize (bf16, contiguous rows): mode 0 act = gelu(a),
// mode 1 act = a * gelu'(b); writes act and the int8 payload / states of act.
cudaError_t launch_act_quantize_rowwise(sb_handle h, int mode, const void* a, const void* b, int64_t rows, int64_t cols,
                                        void* act, int8_t* q, float* state);
// Attention gradients dq / dk / dv [B, H, S, Dh] (bf16, element strides (b, h, s) per tensor in
// `strides`, Dh contiguous) -> packed G [B S x 3 H Dh] and the row-wise int8 payload / states of
// each projection's column block (q[i] [B S x H Dh], st[i] [B S]); cudaErrorNotSupported for
// H Dh > 2048, Dh % 8, or unaligned operands.
cudaError_t launch_heads_pack_quantize(sb_handle h, const void* const* src, const int64_t* strides, int64_t B,
                                       int64_t S, int H, int Dh, void* g, int8_t* const* q, float* const* st);
// y[r, c] += resid[r, c] in place (y, resid bf16 / fp32 of dt, rows x cols contiguous)
cudaError_t launch_add_residual(sb_handle h, void* y, sb_dtype dt, int64_t rows, int64_t cols, const void* resid);
// y[r, c] += bias[c] in place (y is SB_F32 or SB_BF16, rows x cols contiguous)
cudaError_t launch_add_bias(sb_handle h, void* y, sb_dtype dt, int64_t rows, int64_t cols, const float* bias);
cudaError_t launch_fp8_cast(sb_handle h, const float* x, int64_t n, int fmt, float* y);

// gemm_i8.cu
// bias (optional, fp32 [N]): fused into the tensor-core epilogue for bf16 / fp32 outputs,
// otherwise added by launch_add_bias after the product.
// resid (optional, bf16 [M x N], row stride ld_resid; bf16 output only): added in the epilogue.
sb_status gemm_i8(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sb, int scale_mode,
                  int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt, int exact, const float* bias = nullptr,
                  const void* resid = nullptr, int64_t ld_resid = 0);
// gemm_bf16.cu
// Row-wise int8 quantize of G riding along with the dW GEMM (payload q [b x m], row stride ldq
// bytes, states [b]); identical to launch_quantize_rowwise(G).
struct RowQuant {
  int8_t* q;
  int64_t ldq;
  float* state;
};
// rq (optional): also quantize G row-wise — inside the one-wave dW kernel when it applies,
// otherwise as a separate launch before the GEMM.
sb_status wgrad(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n, float* dw,
                int exact, int accumulate, const RowQuant* rq = nullptr);
// dW = G^T X with the epilogue reduce-adding every 32-row block of dW into its owner rank's copy
// of the symmetric buffer holding dw (fused GEMM + reduce-scatter); one-wave bf16 kernel only
// (SB_ERR_UNSUPPORTED otherwise). Every rank's dw must be zeroed (and the zeroing ordered
// before this call on every rank) first.
sb_status wgrad_reduce_scatter(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n,
                               float* dw, const sb_symbuf& sym, const RowQuant* rq);
// True when the one-wave dW kernel (and so wgrad_reduce_scatter) serves an m x n dW over b tokens.
bool dw_wide_serves(sb_handle h, int64_t m, int64_t n, int64_t b);
sb_status matmul_f32_seq(sb_handle h, const float* a, int64_t a_rs, int64_t a_ks, const float* bt, int64_t b_rs,
                         int64_t b_ks, int64_t r, int64_t c, int64_t k, float* y, int accumulate);
sb_status gemm_bf16_tc(sb_handle h, const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K,
                       void* out, sb_dtype out_dt, const float* one);
// gemm_fp8
sb_status gemm_fp8(sb_handle h, const uint8_t* qa, int fa, const float* sa, int axa, const uint8_t* qb, int fb,
                   const float* sb, int axb, int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt);

// dp.cu
// The symmetric buffer holding [p, p + bytes) (nullptr if none).
const sb_symbuf* find_symbuf(sb_handle h, const void* p, size_t bytes);
// Rows [r0, r1) of a rows-row dW owned by `rank` in the fused reduce-scatter: 32-row blocks,
// block rb owned by rank (rb * world) / nblocks (contiguous, sizes differ by at most one block).
void dp_owned_rows(int64_t rows, int rank, int world, int64_t* r0, int64_t* r1);
// Sum all-reduce of n fp32 values in place on `stream` over the handle's communicator (no-op
// without one, or with one rank).
sb_status dp_allreduce_sum_f32(sb_handle h, float* buf, int64_t n, cudaStream_t stream);
// Close every peer mapping and free every symmetric buffer of the handle (sb_destroy).
void dp_free_symmetric(sb_handle h);
// True when the handle has a communicator of more than one rank (or SB_DP_FORCE=1 with one rank,
// which runs the multi-rank code paths against the identity collectives).
bool dp_active(sb_handle h);
// AllQuant int8 dW under token sharding (linear.cpp:239-241): per-feature absmax of G and X maxed
// over ranks, column-wise quantization, raw int32 product summed over ranks as int64, one exact
// dequantization float(double(acc) * s_g * s_x / 16129) into dw (also the int32 scratch).
sb_status dp_allquant_dw(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t n, int64_t m,
                         int8_t* gt_q, float* gt_state, int8_t* xt_q, float* xt_state, unsigned int* words,
                         int64_t* raw64, float* dw);

}  // namespace sb
