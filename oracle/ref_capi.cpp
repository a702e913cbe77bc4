// ref_capi.cpp — extern "C" face of the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. oracle/Makefile compiles this file
// together with the reference's own sources, where they lie under
// /root/reference/proj/core/src (matrix.cpp, quantize.cpp, linear.cpp,
// optimizer.cpp), into oracle/_ref/libref_lowprec.so. Nothing is copied into
// the repo. The library is used for three things only:
//   1. generating tests/golden/ fixtures (tests/golden/make_golden.py),
//   2. pinning oracle/oracle.c against the reference (tests/test_oracle_golden.py),
//   3. the transformer-block parity test (tests/test_block_gpu.py): lowprec::model_forward /
//      model_backward (model.cpp) at depth 1 with identity embedding / head, which is exactly
//      transformer_block + block_backward (model.cpp:287-408) and exposes d(block input),
//   4. bench.py's CPU baseline and `--impl reference` arm: lowprec::linear_forward
//      + lowprec::linear_backward({kSwitchBack, kInt8}) — the reference's own
//      switchback_fwd_bwd unit (bench.cpp:75-81) — on P host threads, each on a
//      token-row shard (rows are independent).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "lowprec/linear.hpp"
#include "lowprec/matrix.hpp"
#include "lowprec/model.hpp"
#include "lowprec/optimizer.hpp"
#include "lowprec/quantize.hpp"

using namespace lowprec;

namespace {
thread_local std::string g_err;

Matrix to_matrix(const float* p, int64_t r, int64_t c) {
  Matrix m(r, c);
  if (r * c) std::memcpy(m.data(), p, size_t(r * c) * sizeof(float));
  return m;
}
void from_matrix(const Matrix& m, float* out) {
  if (m.size()) std::memcpy(out, m.data(), size_t(m.size()) * sizeof(float));
}
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
LinearMode mode_of(int variant, int format) {
  LinearMode m;
  m.variant = LinearVariant(variant);
  m.format = format ? NumericFormat::kFp8 : NumericFormat::kInt8;
  return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_derive_seed(uint64_t seed, uint64_t stream) { return derive_seed(seed, stream); }

int ref_gaussian_matrix(int64_t r, int64_t c, float mean, float stdev, uint64_t seed, float* out) {
  return guarded([&] { from_matrix(gaussian_matrix(r, c, mean, stdev, seed), out); });
}

// axis: 0 row, 1 column, 2 tensor, 3 tensor+transpose (payload is cols x rows)
int ref_quantize_int8(const float* x, int64_t r, int64_t c, int axis, int8_t* q, float* state) {
  return guarded([&] {
    Matrix m = to_matrix(x, r, c);
    QuantizedMatrix qm = axis == 0   ? quantize_rowwise(m)
                         : axis == 1 ? quantize_columnwise(m)
                         : axis == 2 ? quantize_tensorwise(m)
                                     : quantize_tensorwise_transpose(m);
    std::memcpy(q, qm.payload_int8.data(), qm.payload_int8.size());
    std::memcpy(state, qm.state.data(), qm.state.size() * sizeof(float));
  });
}

// fmt: 0 e4m3, 1 e5m2; axis 0 row, 1 column, 2 tensor
int ref_quantize_fp8(const float* x, int64_t r, int64_t c, int fmt, int axis, float* payload,
                     float* state) {
  return guarded([&] {
    QuantizedMatrix qm = quantize_fp8(to_matrix(x, r, c), fmt ? Fp8Format::e5m2() : Fp8Format::e4m3(),
                                      QuantAxis(axis));
    std::memcpy(payload, qm.payload_fp8.data(), qm.payload_fp8.size() * sizeof(float));
    std::memcpy(state, qm.state.data(), qm.state.size() * sizeof(float));
  });
}

int ref_fp8_value_set(int fmt, float* out) {
  std::vector<float> v = fp8_value_set(fmt ? Fp8Format::e5m2() : Fp8Format::e4m3());
  std::memcpy(out, v.data(), v.size() * sizeof(float));
  return int(v.size());
}

int ref_dequantize_int8(const int8_t* q, const float* state, int axis, int64_t r, int64_t c,
                        float* y) {
  return guarded([&] {
    QuantizedMatrix qm;
    qm.rows = r;
    qm.cols = c;
    qm.axis = QuantAxis(axis);
    qm.payload_int8.assign(q, q + r * c);
    size_t ns = axis == 0 ? size_t(r) : axis == 1 ? size_t(c) : 1;
    qm.state.assign(state, state + ns);
    from_matrix(dequantize(qm), y);
  });
}

// y = int8_matmul_dequant(quantize_rowwise(a), quantize_tensorwise(b)) (dual=0)
// or matmul_dequant_dual_rowwise(quantize_rowwise(a), quantize_rowwise(b)) (dual=1)
int ref_int8_matmul(const float* a, const float* b, int64_t r, int64_t c, int64_t k, int dual,
                    float* y) {
  return guarded([&] {
    Matrix ma = to_matrix(a, r, k), mb = to_matrix(b, c, k);
    Matrix out = dual ? matmul_dequant_dual_rowwise(quantize_rowwise(ma), quantize_rowwise(mb))
                      : int8_matmul_dequant(quantize_rowwise(ma), quantize_tensorwise(mb));
    from_matrix(out, y);
  });
}

int ref_matmul(const float* a, const float* bt, int64_t r, int64_t c, int64_t k, float* y) {
  return guarded([&] { from_matrix(matmul(to_matrix(a, r, k), to_matrix(bt, c, k)), y); });
}

// variant: LinearVariant enum order (Standard, SwitchBack, SwitchBackM, SwitchBackQ, AllQuant)
int ref_linear_fwd_bwd(int variant, int format, const float* x, const float* w, const float* g,
                       int64_t b, int64_t n, int64_t m, float* y, float* dx, float* dw) {
  return guarded([&] {
    LinearMode mode = mode_of(variant, format);
    LinearContext ctx;
    Matrix out = linear_forward(mode, to_matrix(x, b, n), to_matrix(w, m, n), &ctx);
    if (y) from_matrix(out, y);
    if (g) {
      auto grads = linear_backward(mode, ctx, to_matrix(g, b, m));
      if (dx) from_matrix(grads.first, dx);
      if (dw) from_matrix(grads.second, dw);
    }
  });
}

// SwitchBack{int8} fwd+bwd on `threads` host threads, token rows split into
// contiguous shards; dW partials summed in shard order. The timed unit of the
// CPU baseline. y/dx/dw may be null (timing only).
int ref_switchback_fwd_bwd_threaded(const float* x, const float* w, const float* g, int64_t b,
                                    int64_t n, int64_t m, int threads, float* y, float* dx,
                                    float* dw) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    if (threads > b) threads = int(b);
    const LinearMode mode = mode_of(1, 0);
    const Matrix wm = to_matrix(w, m, n);
    std::vector<Matrix> partial{size_t(threads)};
    std::vector<std::exception_ptr> errs{size_t(threads)};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int64_t r0 = b * t / threads, r1 = b * (t + 1) / threads;
          LinearContext ctx;
          Matrix xs = to_matrix(x + r0 * n, r1 - r0, n);
          Matrix ys = linear_forward(mode, xs, wm, &ctx);
          auto grads = linear_backward(mode, ctx, to_matrix(g + r0 * m, r1 - r0, m));
          if (y) std::memcpy(y + r0 * m, ys.data(), size_t(ys.size()) * sizeof(float));
          if (dx) std::memcpy(dx + r0 * n, grads.first.data(), size_t(grads.first.size()) * sizeof(float));
          partial[size_t(t)] = std::move(grads.second);
        } catch (...) {
          errs[size_t(t)] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    if (dw) {
      std::memset(dw, 0, size_t(m * n) * sizeof(float));
      for (const Matrix& p : partial)
        for (int64_t i = 0; i < m * n; ++i) dw[i] += p.data()[i];
    }
  });
}

// Two chained SwitchBack int8 linears (the MLP block of model.cpp:324-329 with no activation,
// and its backward, model.cpp:351-360): h = linear_forward(x, w1), y = linear_forward(h, w2),
// (dh, dw2) = linear_backward(ctx2, g), (dx, dw1) = linear_backward(ctx1, dh), with token rows
// sharded over `threads` (every op is per row except the W quantize and the dW sums, whose
// per-thread partials are added in thread order). Outputs may be null.
int ref_switchback_mlp_fwd_bwd_threaded(const float* x, const float* w1, const float* w2, const float* g,
                                        int64_t b, int64_t n, int64_t hd, int64_t m, int threads, float* y,
                                        float* dx, float* dw1, float* dw2) {
  return guarded([&] {
    if (threads < 1) threads = 1;
    if (threads > b) threads = int(b);
    const LinearMode mode = mode_of(1, 0);
    const Matrix w1m = to_matrix(w1, hd, n), w2m = to_matrix(w2, m, hd);
    std::vector<Matrix> p1{size_t(threads)}, p2{size_t(threads)};
    std::vector<std::exception_ptr> errs{size_t(threads)};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          const int64_t r0 = b * t / threads, r1 = b * (t + 1) / threads;
          LinearContext c1, c2;
          const Matrix hs = linear_forward(mode, to_matrix(x + r0 * n, r1 - r0, n), w1m, &c1);
          const Matrix ys = linear_forward(mode, hs, w2m, &c2);
          auto g2 = linear_backward(mode, c2, to_matrix(g + r0 * m, r1 - r0, m));
          auto g1 = linear_backward(mode, c1, g2.first);
          if (y) std::memcpy(y + r0 * m, ys.data(), size_t(ys.size()) * sizeof(float));
          if (dx) std::memcpy(dx + r0 * n, g1.first.data(), size_t(g1.first.size()) * sizeof(float));
          p1[size_t(t)] = std::move(g1.second);
          p2[size_t(t)] = std::move(g2.second);
        } catch (...) {
          errs[size_t(t)] = std::current_exception();
        }
      });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    auto sum = [&](float* dst, const std::vector<Matrix>& parts, int64_t count) {
      if (!dst) return;
      std::memset(dst, 0, size_t(count) * sizeof(float));
      for (const Matrix& p : parts)
        for (int64_t i = 0; i < count; ++i) dst[i] += p.data()[i];
    };
    sum(dw1, p1, hd * n);
    sum(dw2, p2, m * hd);
  });
}

// optimizer_step over `nt` tensors (flat views of shape 1 x numel).
// clipping: 0 none, 1 update_clip, 2 grad_clip. alpha is the (constant) lr_schedule value.
int ref_optimizer_step(int nt, float** theta, const float** grad, float** v, float** u,
                       const int64_t* numel, double alpha, double beta1, double beta2,
                       double beta2_warmup_lambda, double eps, double weight_decay, int clipping,
                       double max_grad_norm, int64_t t, double* out_rms, double* out_eta) {
  return guarded([&] {
    std::vector<Matrix> p, g;
    std::vector<TensorOptState> st;
    st.resize(size_t(nt));
    for (int i = 0; i < nt; ++i) {
      p.push_back(to_matrix(theta[i], 1, numel[i]));
      g.push_back(to_matrix(grad[i], 1, numel[i]));
      st[size_t(i)].v = to_matrix(v[i], 1, numel[i]);
      st[size_t(i)].u = to_matrix(u[i], 1, numel[i]);
    }
    std::vector<TensorRef> refs;
    for (int i = 0; i < nt; ++i) {
      TensorRef r;
      r.name = "t" + std::to_string(i);
      r.param = &p[size_t(i)];
      r.grad = &g[size_t(i)];
      r.state = &st[size_t(i)];
      refs.push_back(r);
    }
    OptimizerHyperparams hp;
    hp.lr_schedule = [alpha](int64_t) { return alpha; };
    hp.beta1 = beta1;
    hp.beta2 = beta2;
    hp.beta2_warmup_lambda = beta2_warmup_lambda;
    hp.eps = eps;
    hp.weight_decay = weight_decay;
    hp.clipping = Clipping(clipping);
    hp.max_grad_norm = max_grad_norm;
    auto infos = optimizer_step(refs, hp, t);
    for (int i = 0; i < nt; ++i) {
      from_matrix(p[size_t(i)], theta[i]);
      from_matrix(st[size_t(i)].v, v[i]);
      from_matrix(st[size_t(i)].u, u[i]);
      if (out_rms) out_rms[i] = infos[size_t(i)].rms;
      if (out_eta) out_eta[i] = infos[size_t(i)].eta;
    }
  });
}

// One pre-norm transformer block forward + backward (model.cpp:287-408) through the public
// model API: depth 1, inputs = I (tokens x tokens) and embed = X^T so the block input is X
// exactly (each output is one product with 1 plus zeros), head = I so logits = block output and
// d(block output) = d_logits; the embed gradient is then d(block input)^T (model.cpp:442+).
// params / grads: norm1.gain, norm1.bias, wq, wk, wv, wo, ls1, ls2, norm2.gain, norm2.bias,
// w1, w2 (12 pointers; ls1 / ls2 ignored without layer scale). y: block output, dx: d(input).
int ref_block_fwd_bwd(int variant, int format, int64_t tokens, int64_t dim, int64_t heads, double mlp_ratio,
                      int layer_scale, const float* const* params, const float* x, const float* d_out, float* y,
                      float* dx, float* const* grads) {
  return guarded([&] {
    ModelConfig cfg;
    cfg.depth = 1;
    cfg.dim = dim;
    cfg.heads = heads;
    cfg.mlp_ratio = mlp_ratio;
    cfg.layer_scale_enabled = layer_scale != 0;
    cfg.linear_mode = mode_of(variant, format);
    cfg.embed_norm = false;
    cfg.input_dim = tokens;
    cfg.output_dim = dim;
    const int64_t hid = cfg.mlp_hidden();
    ModelParams p = zeros_like(cfg);
    const Matrix xm = to_matrix(x, tokens, dim);
    p.embed = xm.transposed();
    for (int64_t i = 0; i < dim; ++i) p.head(i, i) = 1.0f;
    BlockParams& b = p.blocks[0];
    b.norm1.gain = to_matrix(params[0], 1, dim);
    b.norm1.bias = to_matrix(params[1], 1, dim);
    b.wq = to_matrix(params[2], dim, dim);
    b.wk = to_matrix(params[3], dim, dim);
    b.wv = to_matrix(params[4], dim, dim);
    b.wo = to_matrix(params[5], dim, dim);
    if (cfg.layer_scale_enabled) {
      b.ls1 = to_matrix(params[6], 1, dim);
      b.ls2 = to_matrix(params[7], 1, dim);
    }
    b.norm2.gain = to_matrix(params[8], 1, dim);
    b.norm2.bias = to_matrix(params[9], 1, dim);
    b.w1 = to_matrix(params[10], hid, dim);
    b.w2 = to_matrix(params[11], dim, hid);
    Matrix inputs(tokens, tokens);
    for (int64_t i = 0; i < tokens; ++i) inputs(i, i) = 1.0f;
    ModelTape tape;
    const Matrix out = model_forward(cfg, p, inputs, &tape);
    from_matrix(out, y);
    const ModelParams g = model_backward(cfg, p, tape, to_matrix(d_out, tokens, dim));
    from_matrix(g.embed.transposed(), dx);
    const BlockParams& gb = g.blocks[0];
    const Matrix* outs[12] = {&gb.norm1.gain, &gb.norm1.bias, &gb.wq, &gb.wk, &gb.wv, &gb.wo,
                              &gb.ls1,        &gb.ls2,        &gb.norm2.gain, &gb.norm2.bias, &gb.w1, &gb.w2};
    for (int k = 0; k < 12; ++k)
      if (grads[k] && (cfg.layer_scale_enabled || (k != 6 && k != 7))) from_matrix(*outs[k], grads[k]);
  });
}

}  // extern "C"
