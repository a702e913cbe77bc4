/*
 * switchback_b200.h — the C-ABI drop-in boundary of the B200 SwitchBack path.
 *
 * Plain pointers and sizes only (no torch, no C++ types). Device pointers
 * unless an entry point says "host". Every call is stream-ordered on the
 * handle's CUDA stream and returns as soon as the work is enqueued; device-side
 * input errors (non-finite values, which the reference rejects up front) are
 * latched in the handle and reported by sb_synchronize().
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/core). The C++ shim in
 * paper_2304_13013_b200/csrc/lowprec_shim.cpp re-exposes the reference's own
 * lowprec:: signatures (host Matrix in, host Matrix out) on top of this ABI.
 */
#ifndef SWITCHBACK_B200_H
#define SWITCHBACK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SB_ABI_VERSION 1

typedef enum sb_status {
  SB_OK = 0,
  SB_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  SB_ERR_NONFINITE = 2,        /* "non-finite input" (quantize.cpp:11-14, linear.cpp:91-92) */
  SB_ERR_CUDA = 3,
  SB_ERR_UNSUPPORTED = 4
} sb_status;

typedef enum sb_dtype { SB_F32 = 0, SB_BF16 = 1, SB_I32 = 2, SB_I8 = 3, SB_U8 = 4, SB_I64 = 5 } sb_dtype;

/* QuantAxis, quantize.hpp:12 */
typedef enum sb_axis { SB_AXIS_ROW = 0, SB_AXIS_COLUMN = 1, SB_AXIS_TENSOR = 2 } sb_axis;

/* Fp8Format::e4m3() / e5m2(), quantize.hpp:30-31 */
typedef enum sb_fp8_format { SB_E4M3 = 0, SB_E5M2 = 1 } sb_fp8_format;

/* LinearVariant, linear.hpp:23 */
typedef enum sb_variant {
  SB_STANDARD = 0,
  SB_SWITCHBACK = 1,
  SB_SWITCHBACK_M = 2,
  SB_SWITCHBACK_Q = 3,
  SB_ALLQUANT = 4
} sb_variant;

/* NumericFormat, linear.hpp:25 */
typedef enum sb_numeric_format { SB_INT8 = 0, SB_FP8 = 1 } sb_numeric_format;

/* State application of the int8 GEMM epilogue (linear.cpp:54-83). */
typedef enum sb_scale_mode {
  SB_SCALE_ROW_TENSOR = 0, /* int8_matmul_dequant: state_a[i] * state_b / 127^2 (linear.hpp:54) */
  SB_SCALE_ROW_ROW = 1,    /* matmul_dequant_dual_rowwise: state_a[i] * state_b[j] / 127^2 (linear.hpp:58) */
  SB_SCALE_NONE = 2        /* raw integer accumulators (out dtype SB_I32, or SB_I64 beyond k = 133144) */
} sb_scale_mode;

/* Clipping, optimizer.hpp:12-16 */
typedef enum sb_clipping { SB_CLIP_NONE = 0, SB_CLIP_UPDATE = 1, SB_CLIP_GRAD = 2 } sb_clipping;

typedef struct sb_handle_s* sb_handle;

/* ------------------------------------------------------------ runtime -- */
int sb_abi_version(void);
/* Creates a handle bound to `device` (cudaSetDevice semantics) on the default stream. */
sb_status sb_create(int device, sb_handle* out);
sb_status sb_destroy(sb_handle h);
/* `cuda_stream` is a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream). */
sb_status sb_set_stream(sb_handle h, void* cuda_stream);
/* Waits for the handle's stream; returns SB_ERR_NONFINITE (and clears the latch)
 * when a kernel saw a NaN/Inf input since the last call. */
sb_status sb_synchronize(sb_handle h);
/* Non-blocking device error latch (device pointer to one uint32; bit 0 = non-finite). */
uint32_t* sb_error_word(sb_handle h);
/* "<op>: <reason>" — the reference's exception text for the last failure on this thread. */
const char* sb_last_error(void);
/* Kernel launches issued through this handle so far (launch accounting for bench.py). */
uint64_t sb_launch_count(sb_handle h);
/* Tensor-core GEMM tiling for this handle (no reference counterpart: a B200 tuning knob).
 * SB_GEMM_AUTO: 2-CTA (cta_group::2) 256 x 256 tiles when the problem fills the SM pairs,
 * else 1-CTA 128 x 256; the other values force one form (results are identical). */
/* AUTO picks per shape; 1CTA = 128 x 256 tiles; 2CTA = cta_group::2 256 x 256 tiles; WIDE = the
 * transposed cta_group::2 256 x 384 int8 / fp8 kernel (tc_i8_wide.cuh) wherever it applies;
 * 2CTA_MC = the 256 x 256 kernel in clusters of two CTA pairs that share (TMA-multicast) the
 * B operand of vertically adjacent tiles (tc_gemm2.cuh Pipe2<2>). */
typedef enum sb_gemm_path {
  SB_GEMM_AUTO = 0,
  SB_GEMM_1CTA = 1,
  SB_GEMM_2CTA = 2,
  SB_GEMM_WIDE = 3,
  SB_GEMM_2CTA_MC = 4
} sb_gemm_path;
sb_status sb_set_gemm_path(sb_handle h, int path);

/* Device memory + synchronous copies on the handle's stream (for FFI callers without a CUDA runtime). */
sb_status sb_device_alloc(sb_handle h, size_t bytes, void** out);
sb_status sb_device_free(sb_handle h, void* ptr);
sb_status sb_copy_to_device(sb_handle h, void* dst, const void* src, size_t bytes);
sb_status sb_copy_to_host(sb_handle h, void* dst, const void* src, size_t bytes);
/* Matrix::all_finite (matrix.cpp:22-26) as a device check: latches SB_ERR_NONFINITE for sb_synchronize. */
sb_status sb_check_finite(sb_handle h, const void* x, sb_dtype dt, int64_t n);

/* ----------------------------------------------------------- quantize -- */
/* quantize_rowwise, quantize.hpp:67 / quantize.cpp:131-133.
 * x: rows x cols (leading dim ldx elements) of `dt` (SB_F32 or SB_BF16);
 * q: int8 rows x cols (ldq); state: rows floats (absmax, 1.0 for all-zero rows). */
sb_status sb_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                              int8_t* q, int64_t ldq, float* state);

/* quantize_columnwise, quantize.hpp:68 / quantize.cpp:135-137. q (rows x cols, ldq) and/or
 * q_t (cols x rows, ldqt; = quantize_rowwise(x^T), the SwitchBackQ weight path linear.cpp:228-229)
 * may be NULL; state: cols floats. */
sb_status sb_quantize_columnwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state);

/* quantize_tensorwise + quantize_tensorwise_transpose, quantize.hpp:69-71 /
 * quantize.cpp:139-159: one absmax pass, one quantize pass writing q (rows x cols)
 * and/or q_t (cols x rows) from a single read. state: 1 float. */
sb_status sb_quantize_tensorwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                                 int8_t* q, int64_t ldq, int8_t* q_t, int64_t ldqt, float* state);

/* dequantize (int8 branch), quantize.hpp:76 / quantize.cpp:178-197:
 * y = float(double(p) * double(state) / 127). y dtype SB_F32 (bit-exact) or SB_BF16. */
sb_status sb_dequantize(sb_handle h, const int8_t* q, int64_t rows, int64_t cols, int64_t ldq, const float* state,
                        sb_axis axis, void* y, sb_dtype ydt, int64_t ldy);

/* quantize_fp8, quantize.hpp:73 / quantize.cpp:161-176: payload = snap(x / state) with
 * ties to the smaller magnitude, stored as e4m3 / e5m2 bytes (decode = the reference's
 * payload_fp8 value). state: rows / cols / 1 floats per axis. */
sb_status sb_quantize_fp8(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ldx,
                          sb_fp8_format fmt, sb_axis axis, uint8_t* q, int64_t ldq, float* state);

/* dequantize (fp8 branch), quantize.cpp:185-189: y = float(double(value(p)) * double(state)). */
sb_status sb_dequantize_fp8(sb_handle h, const uint8_t* q, int64_t rows, int64_t cols, int64_t ldq, sb_fp8_format fmt,
                            const float* state, sb_axis axis, void* y, sb_dtype ydt, int64_t ldy);

/* fp8_cast, quantize.hpp:44 / quantize.cpp:78-84: y = nearest e4m3/e5m2 value of x, ties to the
 * smaller magnitude, saturating at the format's largest finite value. */
sb_status sb_fp8_cast(sb_handle h, const float* x, int64_t n, sb_fp8_format fmt, float* y);

/* dequantize (fp8 branch) over DECODED payload values p (fp32 value-set members, the reference's
 * payload_fp8 representation): y = float(double(p) * double(state)), quantize.cpp:185-189. */
sb_status sb_dequantize_values(sb_handle h, const float* p, int64_t rows, int64_t cols, const float* state, sb_axis axis,
                               float* y);

/* transpose_tensorwise's payload move (linear.cpp:170-189): out[cols x rows] = in[rows x cols]^T. */
sb_status sb_transpose_i8(sb_handle h, const int8_t* in, int64_t rows, int64_t cols, int8_t* out);

/* Bias gradient of the nn module's linears (no reference counterpart: the reference's linears
 * carry no bias, model.cpp:324-329): out[c] = sum over rows of x[r, c] in fp32, x bf16 or fp32
 * with leading dim ld >= cols. Deterministic (fixed split and summation order for a given shape
 * and device); rows == 0 writes zeros. Uses the stream's internal scratch (<= 1 MB). */
sb_status sb_column_sums(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols, int64_t ld, float* out);

/* --------------------------------------------------------------- GEMM -- */
/* int8_matmul_dequant / matmul_dequant_dual_rowwise, linear.hpp:54-58 / linear.cpp:39-83.
 * out[M x N] (ld N) = (qa[M x K] . qb[N x K]^T) with the state epilogue of `mode`.
 * Both operands K-major (row-major, leading dim K). Output dtype:
 *   SB_F32 + exact=1 : float(double(acc) * sa_i * sb_j / 16129.0), bit-identical to linear.cpp:49
 *   SB_F32 + exact=0 : same formula in fp32
 *   SB_BF16          : fp32 formula rounded to bf16 (the performance path)
 *   SB_I32 / SB_I64  : raw accumulators (mode must be SB_SCALE_NONE) */
sb_status sb_gemm_i8(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sb,
                     sb_scale_mode mode, int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt, int exact);

/* sb_gemm_i8 with the layer epilogue: y = dequant(acc) (+ bias[N], fp32) (+ resid[M x N] of the
 * output dtype, leading dim ld_resid), each added in fp32 before the single output rounding.
 * bias / resid may be NULL. Serves grouped projections (model.cpp:303-305: q / k / v as one
 * GEMM whose per-column W scale is its projection's, mode SB_SCALE_ROW_ROW) and the summed
 * input gradients of such a group (dX = dX_q + dX_k + dX_v, the residual carrying the sum). */
sb_status sb_gemm_i8_epilogue(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sb,
                              sb_scale_mode mode, int64_t M, int64_t N, int64_t K, const float* bias,
                              const void* resid, int64_t ld_resid, void* out, sb_dtype out_dt, int exact);

/* matmul, matrix.hpp:51 / matrix.cpp:53-68: y[r x c] = a[r x k] . bt[c x k]^T with a strictly
 * sequential fp32 reduction per output and no FMA — bit-identical to the reference. */
sb_status sb_matmul_f32(sb_handle h, const float* a, const float* bt, int64_t r, int64_t c, int64_t k, float* y);

/* wgrad_full_precision, linear.cpp:193-195: dw[m x n] (+)= g[b x m]^T . x[b x n].
 *   exact=1 (SB_F32 in): sequential fp32 over the b tokens, bit-identical to the reference.
 *   exact=0 (SB_BF16 in): bf16 tcgen05 GEMM reading g and x in place (MN-major), fp32 out.
 * accumulate=1 adds into dw (fp32) instead of overwriting. */
sb_status sb_wgrad(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n,
                   float* dw, int exact, int accumulate);
/* The SwitchBack backward's two consumers of G in one launch (linear.cpp:232-245 reads G for
 * quantize_rowwise(G) -> dX and for wgrad_full_precision(G, X) -> dW): dw[m x n] = g^T x as
 * sb_wgrad (exact=0, no accumulate), and g_q[b x m] (row stride ldq bytes) / g_state[b] =
 * sb_quantize_rowwise(g), bit for bit. On the one-wave bf16 dW kernel the quantize runs in its
 * otherwise idle warps while the tensor cores stream the GEMM; elsewhere it is a separate launch
 * before the GEMM. Replaces the pair quantize_rowwise(grad_output) + wgrad_full_precision
 * issued by linear_backward (linear.cpp:232, :245). */
sb_status sb_wgrad_quantize_rowwise(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                    int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state);

/* fp8 GEMM (the SwitchBack fp8 simulation, linear.cpp:148-153 / :250-266): out = (qa . qb^T)
 * * sa_i * sb_j with qa/qb e4m3|e5m2 bytes, K-major; states per row (row axis) or broadcast
 * (tensor axis). Tensor-core accumulation (fp32) — tolerance parity. */
sb_status sb_gemm_fp8(sb_handle h, const uint8_t* qa, sb_fp8_format fa, const float* sa, sb_axis axa,
                      const uint8_t* qb, sb_fp8_format fb, const float* sb, sb_axis axb, int64_t M, int64_t N,
                      int64_t K, void* out, sb_dtype out_dt);

/* ------------------------------------------------------------- layer ---- */
/* LinearMode, linear.hpp:30-35. exact = 1 selects the reference-bit-exact numerics
 * (fp32 I/O, fp64 dequant epilogue, sequential fp32 weight gradient); exact = 0 is the
 * B200 performance path (bf16 I/O, tcgen05 int8 + bf16 GEMMs, fp32 dW). */
typedef struct sb_linear_mode {
  int32_t variant;      /* sb_variant */
  int32_t format;       /* sb_numeric_format */
  int32_t fp8_forward;  /* sb_fp8_format, default SB_E4M3 */
  int32_t fp8_gradient; /* sb_fp8_format, default SB_E5M2 */
  int32_t exact;
} sb_linear_mode;

/* LinearContext, linear.hpp:39-48. Filled by sb_linear_forward; consumed by
 * sb_linear_backward. Unlike the reference (deep copies, linear.cpp:140-143) it
 * references the caller's x and w, which must stay alive and unmodified until
 * the backward; quantized tensors live in the caller's workspace. */
typedef struct sb_linear_ctx {
  sb_linear_mode mode;
  int64_t b, n, m;
  sb_dtype dt;
  const void* x; /* b x n */
  const void* w; /* m x n */
  int8_t* w_q_t; /* cached W_int8^T (n x m, tensor-wise), reused by the backward */
  float* w_state;
  int8_t* x_q; /* SwitchBackM: saved X_int8 (b x n) + row states */
  float* x_state;
  void* workspace;
  size_t workspace_bytes;
  int32_t valid;
} sb_linear_ctx;

/* Workspace the forward+backward pair needs (caller allocates once, reuses). */
sb_status sb_linear_workspace_size(const sb_linear_mode* mode, int64_t b, int64_t n, int64_t m, size_t* bytes);

/* Byte offsets, inside a linear workspace, of the quantized operands the layer writes there
 * (the reference's QuantizedMatrix temporaries, linear.cpp:134 / :234-235): X's row-wise
 * payload [b x n] and states [b]; W's payload [m x n] (tensor-wise, or row-wise for
 * SwitchBackQ) and its transpose [n x m]; W's state(s); G's row-wise payload [b x m] and
 * states [b] (written by sb_linear_backward unless G came prequantized). Lets a caller (or a
 * parity test) read the layer's own int8 operands without re-quantizing. */
typedef struct sb_linear_ws_layout {
  size_t x_q, x_state, w_q, w_q_t, w_state, g_q, g_state, total;
} sb_linear_ws_layout;
sb_status sb_linear_workspace_layout(const sb_linear_mode* mode, int64_t b, int64_t n, int64_t m,
                                     sb_linear_ws_layout* out);

/* linear_forward, linear.hpp:62-63 / linear.cpp:113-164: y[b x m] = X W^T through the
 * variant's quantized path. x/w/y are `dt` (SB_F32 or SB_BF16). ctx may be NULL. */
sb_status sb_linear_forward(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w, sb_dtype dt,
                            int64_t b, int64_t n, int64_t m, void* y, sb_linear_ctx* ctx, void* workspace,
                            size_t workspace_bytes);

/* sb_linear_forward plus an fp32 per-output-column bias (m values, NULL = none): y = X W^T + b.
 * The reference applies biases outside linear_forward (model.cpp:303-333); here the add is
 * fused into the int8 GEMM epilogue (one rounding to dt, no extra pass over y). */
sb_status sb_linear_forward_bias(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                 const float* bias, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                                 sb_linear_ctx* ctx, void* workspace, size_t workspace_bytes);

/* linear_backward, linear.hpp:66-67 / linear.cpp:199-278: {dx [b x n] (dt), dw [m x n] (fp32)}.
 * dw_accumulate = 1 adds into dw (gradient accumulation / DP bucket). */
sb_status sb_linear_backward(sb_handle h, const sb_linear_mode* mode, const sb_linear_ctx* ctx, const void* g,
                             void* dx, float* dw, int dw_accumulate);

/* ---- producer fusion (no reference counterpart: the reference
 * quantizes inside linear_forward / linear_backward, linear.cpp:130-134, 216-235) ----
 * act = gelu(pre) (erf form) written as bf16 together with its row-wise int8 payload and
 * states: the payload/states equal sb_quantize_rowwise(act) bit for bit. */
sb_status sb_gelu_quantize_rowwise(sb_handle h, const void* pre, sb_dtype dt, int64_t rows, int64_t cols, void* act,
                                   int8_t* q, float* state);
/* g = dact * gelu'(pre) as bf16 plus its row-wise int8 payload and states. */
sb_status sb_gelu_backward_quantize_rowwise(sb_handle h, const void* dact, const void* pre, sb_dtype dt, int64_t rows,
                                            int64_t cols, void* g, int8_t* q, float* state);
/* Producer fusion at the q/k/v projection's backward (model.cpp:303-305, 385-397): the attention
 * gradients dq, dk, dv arrive head-major [B, H, S, Dh] (bf16; strides[3 i + 0/1/2] = element
 * strides of b, h, s of tensor i; Dh contiguous). One pass writes the packed output gradient
 * g [B S x 3 H Dh] that the grouped dW GEMM reads and, from the same registers, each projection's
 * row-wise int8 payload q[i] [B S x H Dh] / states state[i] [B S] — equal to quantize_rowwise of
 * g's column block i (the three per-projection quantizations of the grouped backward). */
sb_status sb_heads_pack_quantize(sb_handle h, const void* const* dqkv, const int64_t* strides, int64_t B, int64_t S,
                                 int H, int Dh, void* g, int8_t* const* q, float* const* state);

/* out = LayerNorm(x) (over each row of cols; fp32 gamma, beta; bf16 x and out) with its row-wise
 * int8 payload and states, plus per-row mean and rstd (fp32) for the backward. Rows of up to
 * 2048 columns (multiple of 8); SB_ERR_UNSUPPORTED otherwise. */
sb_status sb_layernorm_quantize_rowwise(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                        const float* gamma, const float* beta, float eps, void* out, int8_t* q,
                                        float* state, float* mean, float* rstd);
/* LayerNorm backward for the fused pre-norm path: dx (bf16), dgamma, dbeta (fp32, may be NULL)
 * from dh, x (bf16) and the forward's mean / rstd; deterministic (fixed-order column sums).
 * Rows of up to 1280 columns; workspace from sb_layernorm_backward_workspace_size. */
sb_status sb_layernorm_backward_workspace_size(sb_handle h, int64_t cols, size_t* bytes);
sb_status sb_layernorm_backward(sb_handle h, const void* dh, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                const float* mean, const float* rstd, const float* gamma, void* dx, float* dgamma,
                                float* dbeta, void* workspace, size_t workspace_bytes);
/* sb_linear_forward_bias with X already quantized row-wise by its producer (x_q b x n, x_state b):
 * int8 SwitchBack / SwitchBackM / SwitchBackQ, non-exact. x stays referenced by ctx (dW). */
sb_status sb_linear_forward_prequant(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                                     const float* x_state, const void* w, const float* bias, sb_dtype dt, int64_t b,
                                     int64_t n, int64_t m, void* y, sb_linear_ctx* ctx, void* workspace,
                                     size_t workspace_bytes);
/* y = residual + (X W^T + bias): the residual (dt, b x m, contiguous) is added in the int8 GEMM
 * epilogue before the single rounding to dt (the block's skip connection, model.cpp:327-333).
 * x_q / x_state may be NULL (X quantized here) or a producer's payload as in _prequant. */
sb_status sb_linear_forward_residual(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                                     const float* x_state, const void* w, const float* bias, const void* residual,
                                     sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y, sb_linear_ctx* ctx,
                                     void* workspace, size_t workspace_bytes);
/* linear_forward with every optional producer-side input at once (each may be NULL):
 *   x_q / x_state  X already quantized row-wise by its producer (LayerNorm / GELU fusion);
 *   w_absmax       W's tensor-wise absmax as an fp32-bit-pattern word, as sb_stableadamw_step_ex
 *                  writes it next to the bf16 shadow weight: W is quantized in one pass;
 *   bias, residual as sb_linear_forward_bias / _residual.
 * Prequantized X needs a row-wise int8 variant (SwitchBack, SwitchBackM, SwitchBackQ); w_absmax
 * a tensor-wise one (SwitchBack, SwitchBackM). */
sb_status sb_linear_forward_ex(sb_handle h, const sb_linear_mode* mode, const void* x, const int8_t* x_q,
                               const float* x_state, const void* w, const unsigned int* w_absmax, const float* bias,
                               const void* residual, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                               sb_linear_ctx* ctx, void* workspace, size_t workspace_bytes);

/* sb_linear_backward with G already quantized row-wise by its producer (g_q b x m, g_state b). */
sb_status sb_linear_backward_prequant(sb_handle h, const sb_linear_mode* mode, const sb_linear_ctx* ctx, const void* g,
                                      const int8_t* g_q, const float* g_state, void* dx, float* dw, int dw_accumulate);

/* The reference bench's `switchback_fwd_bwd` unit (bench.cpp:75-81) over HOST buffers:
 * copies x (b x n), w (m x n), g (b x m) in, runs forward + backward, copies y, dx, dw
 * out. Token rows are pipelined in chunks across two streams so PCIe copies overlap
 * the kernels. dt applies to x, w, g, y, dx; dw is fp32. Host buffers should be pinned. */
sb_status sb_switchback_fwd_bwd_host(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                     const void* g, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y, void* dx,
                                     float* dw);

/* Asynchronous form: enqueues the same pipeline and returns; y, dx, dw (and the host inputs)
 * must stay untouched until sb_host_pipeline_wait(h). Consecutive calls alternate between two
 * device pools, so one call's uploads overlap the previous call's drain (a multi-layer step
 * keeps both PCIe directions busy end to end). */
sb_status sb_switchback_fwd_bwd_host_async(sb_handle h, const sb_linear_mode* mode, const void* x, const void* w,
                                           const void* g, sb_dtype dt, int64_t b, int64_t n, int64_t m, void* y,
                                           void* dx, float* dw);
/* Activation between the two linears of sb_switchback_mlp_fwd_bwd_host. */
typedef enum sb_activation { SB_ACT_NONE = 0, SB_ACT_GELU = 1 } sb_activation;

/* The MLP block of the reference's transformer_block (model.cpp:324-329) and its backward
 * (model.cpp:351-360) over HOST buffers: two chained SwitchBack int8 linears
 *   h_pre = linear_forward(x, w1) (b x hd), h = act(h_pre), y = linear_forward(h, w2) (b x m);
 *   (d_h, dw2) = linear_backward(w2_ctx, g), d_hpre = d_h * act'(h_pre),
 *   (dx, dw1) = linear_backward(w1_ctx, d_hpre).
 * x (b x n), w1 (hd x n), w2 (m x hd), g (b x m) in; y (b x m), dx (b x n) out in dt, dw1 / dw2
 * fp32. The hidden activation and its gradient never leave the device: token chunks stream
 * through (H2D | kernels | D2H overlapped), so PCIe carries only the block's inputs and outputs.
 * activation: SB_ACT_NONE (the two linears back to back) or SB_ACT_GELU (bf16, not exact;
 * gelu(double) rounded to float as model.cpp:327, fused into the quantize kernels). Y and dX
 * are per-row and bit-identical to the device-resident path; dw1 / dw2 sum the chunks in order.
 * With a communicator on the handle (sb_dp_init, world > 1) each rank passes its own token shard
 * and dw1 / dw2 come back summed over the ranks (NCCL all-reduce on the device before the copy). */
sb_status sb_switchback_mlp_fwd_bwd_host(sb_handle h, const sb_linear_mode* mode, int activation, const void* x,
                                         const void* w1, const void* w2, const void* g, sb_dtype dt, int64_t b,
                                         int64_t n, int64_t hd, int64_t m, void* y, void* dx, float* dw1, float* dw2);
/* Asynchronous form (same pools / rules as sb_switchback_fwd_bwd_host_async). */
sb_status sb_switchback_mlp_fwd_bwd_host_async(sb_handle h, const sb_linear_mode* mode, int activation, const void* x,
                                               const void* w1, const void* w2, const void* g, sb_dtype dt, int64_t b,
                                               int64_t n, int64_t hd, int64_t m, void* y, void* dx, float* dw1,
                                               float* dw2);
/* Waits for every enqueued host-pipeline call; reports non-finite inputs like sb_synchronize. */
sb_status sb_host_pipeline_wait(sb_handle h);

/* --------------------------------------------------------- optimizer ---- */
/* TensorRef, optimizer.hpp:74-79 (device pointers, fp32, numel elements each). */
typedef struct sb_adamw_tensor {
  float* theta;
  const float* grad;
  float* v;
  float* u;
  int64_t numel;
} sb_adamw_tensor;

/* OptimizerHyperparams, optimizer.hpp:21-33, with alpha = lr_schedule(t) evaluated by the
 * caller (the reference evaluates its host std::function, optimizer.cpp:114). */
typedef struct sb_adamw_hparams {
  double alpha;
  double beta1;
  double beta2;
  double beta2_warmup_lambda; /* > 0 selects beta2_warmup (optimizer.cpp:44-49) */
  double eps;
  double weight_decay;
  double max_grad_norm; /* kGradClip only */
  int32_t clipping;     /* sb_clipping */
} sb_adamw_hparams;

sb_status sb_stableadamw_workspace_size(const sb_adamw_tensor* tensors, int ntensors, size_t* bytes);

/* optimizer_step, optimizer.hpp:85-86 / optimizer.cpp:102-172. `tensors` is a HOST array.
 * rms_out / eta_out: DEVICE arrays of ntensors doubles (TensorStepInfo, optimizer.hpp:69-72),
 * may be NULL. Element math in fp64 mirroring optimizer.cpp:142-146,162-167. */
sb_status sb_stableadamw_step(sb_handle h, const sb_adamw_tensor* tensors, int ntensors, const sb_adamw_hparams* hp,
                              int64_t t, double* rms_out, double* eta_out, void* workspace, size_t workspace_bytes);

/* The trainer's gradient-to-update path (trainer.cpp:127-155) in the optimizer's own passes:
 *   filter_nonfinite (optimizer.cpp:83-100): g' = f32(double(g) / loss_scale) formed on the fly
 *     (the gradient buffers are not rewritten); a tensor with a non-finite g' is skipped — its
 *     theta / v / u stay untouched, rms = NaN, eta = 0 — and with per_tensor_skip = 0 one bad
 *     tensor skips them all;
 *   grad_absmax (trainer.cpp:138): max |g'| per tensor (NaN ignored, as Matrix::abs_max);
 *   the in-step global-norm clip (optimizer.cpp:121-131) over the tensors that are applied;
 * and, for the NEXT step's forward, the weight's bf16 shadow copy and its tensor-wise absmax
 * (the quantize_tensorwise state, quantize.cpp:139-141) written by the theta update itself
 * (optimizer.cpp:162-167), so the next forward quantizes W without its own absmax pass
 * (sb_quantize_tensorwise_from_absmax, sb_linear_forward_ex). One read-only statistics pass
 * over g runs first when skipping, telemetry or the global-norm clip needs it (the skip
 * decision must precede any state update); every other pass is the plain step's. */
typedef struct sb_adamw_extras {
  double loss_scale;              /* LossScaler::scale (> 0); 1 = no unscaling */
  int32_t per_tensor_skip;        /* LossScaler::per_tensor_skip */
  int32_t* skipped;               /* DEVICE [ntensors] out: 1 = skipped this step (or NULL) */
  float* grad_absmax;             /* DEVICE [ntensors] out (or NULL) */
  void* const* shadow_bf16;       /* HOST [ntensors] of DEVICE bf16 pointers (entries may be NULL) */
  unsigned int* const* absmax_word; /* HOST [ntensors] of DEVICE words: max |bf16(theta')| as fp32 bits */
} sb_adamw_extras;

sb_status sb_stableadamw_step_ex(sb_handle h, const sb_adamw_tensor* tensors, int ntensors,
                                 const sb_adamw_hparams* hp, int64_t t, const sb_adamw_extras* extras,
                                 double* rms_out, double* eta_out, void* workspace, size_t workspace_bytes);

/* ZeRO-1 StableAdamW: `tensors[i]` is this rank's contiguous shard of tensor i
 * (e.g. the dW rows it owns after sb_wgrad_reduce_scatter, with theta / v / u rows to match) and
 * numel_total[i] the whole tensor's element count. RMS couples a whole tensor
 * (optimizer.cpp:148-157), so the step splits there:
 *   phase 1: v, u of the shard, and per tensor the shard's sum of g^2 / max(u, eps^2) (fp64,
 *            fixed order) into shard_sums (DEVICE [ntensors]);
 *   (the caller sums shard_sums over ranks: one fp64 all-reduce of ntensors values)
 *   phase 2: RMS = sqrt(total / numel_total), eta, the theta update of the shard; optional bf16
 *            shadow rows + tensor-wise absmax words for the next forward, as sb_stableadamw_step_ex.
 * sb_stableadamw_step_sharded runs both with sb_dp_allreduce_sum_f64 between them (the handle's
 * communicator; one rank: no collective) and max-reduces the absmax words over ranks afterwards
 * (sb_dp_allreduce_max_words: a shard's word covers its rows only; with the split entries the
 * caller does that max). v, u are bitwise the unsharded step's; RMS differs only by
 * the cross-rank summation order (theta bitwise when eta does not depend on it, e.g. RMS <= 1
 * under update clipping). Plain steps: kGradClip is refused (it needs the global norm).
 * Workspace: sb_stableadamw_sharded_workspace_size. HOST arrays: tensors, numel_total,
 * shadow_bf16, absmax_word (may be NULL). */
sb_status sb_stableadamw_sharded_workspace_size(const sb_adamw_tensor* tensors, int ntensors, size_t* bytes);
sb_status sb_stableadamw_shard_phase1(sb_handle h, const sb_adamw_tensor* tensors, const int64_t* numel_total,
                                      int ntensors, const sb_adamw_hparams* hp, int64_t t, double* shard_sums,
                                      void* workspace, size_t workspace_bytes);
sb_status sb_stableadamw_shard_phase2(sb_handle h, const sb_adamw_tensor* tensors, const int64_t* numel_total,
                                      int ntensors, const sb_adamw_hparams* hp, int64_t t, const double* total_sums,
                                      void* const* shadow_bf16, unsigned int* const* absmax_word, double* rms_out,
                                      double* eta_out, void* workspace, size_t workspace_bytes);
sb_status sb_stableadamw_step_sharded(sb_handle h, const sb_adamw_tensor* tensors, const int64_t* numel_total,
                                      int ntensors, const sb_adamw_hparams* hp, int64_t t, void* const* shadow_bf16,
                                      unsigned int* const* absmax_word, double* rms_out, double* eta_out,
                                      void* workspace, size_t workspace_bytes);

/* quantize_tensorwise (+ transpose) of x with its absmax already known (an fp32-bit-pattern word
 * as sb_stableadamw_step_ex writes it): one pass, payloads bit-identical to sb_quantize_tensorwise. */
sb_status sb_quantize_tensorwise_from_absmax(sb_handle h, const void* x, sb_dtype dt, int64_t rows, int64_t cols,
                                             int64_t ldx, const unsigned int* absmax_word, int8_t* q, int64_t ldq,
                                             int8_t* q_t, int64_t ldqt, float* state);

/* compute_rms, optimizer.hpp:54 / optimizer.cpp:31-42: *out (DEVICE double) =
 * sqrt(mean(g^2 / max(u, eps^2))), fp64, fixed-order reduction. */
sb_status sb_compute_rms(sb_handle h, const float* g, const float* u, int64_t n, double eps, double* out);

/* grad_clip_global_norm, optimizer.hpp:59 / optimizer.cpp:72-81: scales every gradient by
 * max_norm / norm when the global L2 norm exceeds max_norm. `grads` / `numel` are HOST arrays
 * of device pointers / sizes. */
sb_status sb_grad_clip_global_norm(sb_handle h, float* const* grads, const int64_t* numel, int n, double max_norm);

/* filter_nonfinite, optimizer.hpp:67 / optimizer.cpp:83-100: out_i = float(double(g_i) / scale);
 * skipped[i] (DEVICE int32) = 1 when out_i has a non-finite entry; with per_tensor_skip = 0 any
 * bad tensor marks all of them. */
sb_status sb_filter_nonfinite(sb_handle h, const float* const* grads, float* const* out, const int64_t* numel, int n,
                              double scale, int per_tensor_skip, int32_t* skipped);

/* ------------------------------------------------- data parallelism (dp.cu) -- */
/* Token-dimension data parallelism, one process per GPU. The library opens
 * libnccl.so.2 at run time. Setup as NCCL's own: rank 0 gets a 128-byte id, every rank receives
 * it out of band and calls sb_dp_init on its handle. */
sb_status sb_dp_available(int* nccl_version); /* SB_ERR_UNSUPPORTED without libnccl.so.2 */
sb_status sb_dp_unique_id(uint8_t* id_out /* 128 bytes */);
sb_status sb_dp_init(sb_handle h, const uint8_t* id, int rank, int world);
sb_status sb_dp_rank(sb_handle h, int* rank, int* world);
/* dW all-reduce (sum, in place) of n device fp32 buffers, on the handle's communication stream
 * after the work already enqueued on its stream; returns at once (overlaps the next layer's
 * backward). `bufs` / `numel` are HOST arrays. sb_dp_wait joins it back into the stream. */
sb_status sb_dp_allreduce_grads_async(sb_handle h, float* const* bufs, const int64_t* numel, int n);
sb_status sb_dp_wait(sb_handle h);
/* Stream-ordered small all-reduces: max of uint32 absmax words (AllQuant's token-dimension
 * scales across ranks, linear.cpp:239-241) and sum of doubles (a sharded optimizer's RMS sums). */
sb_status sb_dp_allreduce_max_u32(sb_handle h, unsigned int* words, int64_t n);
sb_status sb_dp_allreduce_sum_f64(sb_handle h, double* vals, int64_t n);
/* Max all-reduce of n separate device uint32 words (`words` is a HOST array of device pointers,
 * entries may be NULL), one NCCL group. */
sb_status sb_dp_allreduce_max_words(sb_handle h, unsigned int* const* words, int n);
sb_status sb_dp_destroy(sb_handle h);

/* Fused dW GEMM + reduce-scatter over peer memory (SURVEY.md §8e stage 2). dW lives in a
 * symmetric buffer: the same allocation on every rank, each rank's copy mapped into every
 * process (CUDA IPC over NVLink). The one-wave dW kernel's epilogue reduce-adds (TMA
 * cp.reduce.async.bulk .add.f32) every 32-row block of G_r^T X_r into the copy of the rank owning
 * that block (sb_dp_owned_rows), so the reduction streams out while the GEMM runs; the owned rows
 * are then all-gathered. The sum order across ranks is not fixed: dW matches the single-GPU
 * result within fp32 tolerance (with one rank: bit-identical to sb_wgrad).
 *   alloc:    cudaMalloc + cudaIpcGetMemHandle (64-byte handle out);
 *   open:     map the peers' copies from the world x 64 bytes of handles (exchanged out of band);
 *   exchange: alloc's handle all-gathered over the handle's NCCL communicator, then open. */
sb_status sb_dp_symmetric_alloc(sb_handle h, size_t bytes, void** ptr, uint8_t* ipc_handle /* 64 bytes */);
sb_status sb_dp_symmetric_open(sb_handle h, void* ptr, int rank, int world, const uint8_t* ipc_handles);
sb_status sb_dp_symmetric_exchange(sb_handle h, void* ptr, const uint8_t* ipc_handle);
sb_status sb_dp_symmetric_free(sb_handle h, void* ptr);
/* Rows [r0, r1) of a `rows`-row dW that `rank` owns: 32-row blocks, block rb -> rank rb*world/nblocks. */
sb_status sb_dp_owned_rows(int64_t rows, int rank, int world, int64_t* r0, int64_t* r1);
/* The fused GEMM alone: dw (m x n fp32, inside an opened symmetric buffer) must be zeroed on every
 * rank, and that ordered before this call on every rank (sb_dp_barrier). g_q / g_state (optional):
 * G's row-wise quantize in the same launch, as sb_wgrad_quantize_rowwise. bf16 operands, shapes
 * the one-wave dW kernel serves (SB_ERR_UNSUPPORTED otherwise). */
sb_status sb_wgrad_reduce_scatter(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                  int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state);
/* Stream-ordered barrier over the communicator (a one-element all-reduce). */
sb_status sb_dp_barrier(sb_handle h);
/* Every owner's rows of dw broadcast into the other ranks' copies (one NCCL group). */
sb_status sb_dp_allgather_rows(sb_handle h, float* dw, int64_t m, int64_t n);
/* zero + barrier + sb_wgrad_reduce_scatter + barrier + sb_dp_allgather_rows on the handle's
 * stream: dw = sum over ranks of G_r^T X_r on every rank. Shapes the one-wave dW kernel does not
 * serve (e.g. a 1280 x 1280 out-projection) take the local dW GEMM + a NCCL sum all-reduce instead,
 * with the same result contract; dw must still lie in a symmetric buffer. */
sb_status sb_dp_wgrad_allreduce_fused(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m,
                                      int64_t n, float* dw, int8_t* g_q, int64_t ldq, float* g_state);

#ifdef __cplusplus
}
#endif
#endif /* SWITCHBACK_B200_H */
