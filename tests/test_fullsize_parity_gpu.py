"""Full-size parity at every BASELINE.json config, on ALL rows.

For each linear of configs 1-4 at its full token count the layer runs on the B200 and:

* the int8 payloads and scales the layer itself wrote (X row-wise, W tensor-wise and its
  transpose, read out of the layer's workspace through the context pointers) and G's row-wise
  payload are compared BIT FOR BIT with the C oracle (oracle/oracle.c, pinned against the
  reference) run over the whole tensor on the host;
* the raw int32 accumulators of the forward and dX GEMMs are compared bit for bit, over the
  whole output, with an fp64 GPU matmul of the ORACLE's payloads (exact: every partial sum is
  an integer below 2^53; linear.cpp:43-48);
* Y and dX (bf16) are compared, element by element on the whole tensor, with the reference's
  dequant formula f32(double(acc) * s_a * s_b / 16129) (linear.cpp:49) evaluated in fp64 from
  the oracle's payloads and scales: |y - ref| <= 2^-8 |ref| (bf16 rounding of the fp32
  epilogue; the BASELINE tolerance is 1e-2 relative, this is ~40x tighter);
* dW (fp32, bf16 operands, K = T) is compared on the whole tensor with the fp64 product
  G^T X: ||dW - ref|| / ||ref|| < 2e-4, and every element within 1e-3 of sqrt(sum_t g^2 x^2).

Config 1 also runs in exact mode, where Y and dX must equal the reference's fp64 epilogue
bit for bit on every element, and dW rows equal the reference's sequential fp32 loop.
Config 5 checks v / u / theta bitwise on a full ViT-H block's tensor set (19.66 M params).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L
from tests._util import fp8_decode

pytestmark = pytest.mark.gpu

T_VIT = 256 * 257  # 65792 tokens: 256 images x 257 tokens (BASELINE configs 2-4)

# (config, T, n, m): every linear the BASELINE configs name
LINEARS = [
    ("c1", 8192, 1024, 4096),
    ("c2_fc1", T_VIT, 1280, 5120),
    ("c2_fc2", T_VIT, 5120, 1280),
    ("c3_qkv", T_VIT, 1280, 3840),
    ("c3_out", T_VIT, 1280, 1280),
]


def _inputs(T, n, m, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(T, n, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(m, n, device="cuda", generator=g) * n ** -0.5).to(torch.bfloat16)  # model.cpp:199-202
    gr = torch.randn(T, m, device="cuda", generator=g).to(torch.bfloat16)
    x[3] = 0  # zero row: sentinel scale 1.0 (quantize.cpp:98-99)
    x[5, ::7] *= 100  # outlier columns
    gr[T - 1] = 0
    return x, w, gr


def _host_f32(t):
    return t.float().cpu().numpy()


def _oracle_q(a_f32, axis):
    q, s = O.quantize(a_f32, axis)
    return torch.from_numpy(q).cuda(), torch.from_numpy(s).cuda()


def _exact_raw(qa, qb):
    """sum_k qa[i,k] qb[j,k] in fp64 on the GPU: exact (|sum| <= 127^2 K < 2^53)."""
    return qa.double() @ qb.double().T


def _dequant_ref(raw, sa, sb):
    """linear.cpp:49: float(double(acc) * sa_i * sb_j / 16129.0), left to right. The divisor is
    a full tensor: torch turns division by a Python scalar into a multiply by its reciprocal."""
    t = (raw * sa.double()[:, None]) * sb.double()[None, :]
    return (t / torch.full_like(t, 16129.0)).float()


def _assert_bf16_close(got, ref, what):
    err = (got.float() - ref).abs()
    bound = ref.abs() * 2.0 ** -8 + 1e-30
    bad = int((err > bound).sum())
    assert bad == 0, f"{what}: {bad} elements beyond 2^-8 relative (max err {err.max().item():.3e})"
    rel = (torch.linalg.vector_norm((got.float() - ref).double()) / torch.linalg.vector_norm(ref.double())).item()
    assert rel < 1e-2, f"{what}: relative error {rel}"


def _assert_dw(dw, g, x, what):
    ref = g.double().T @ x.double()
    rel = (torch.linalg.vector_norm(dw.double() - ref) / torch.linalg.vector_norm(ref)).item()
    assert rel < 2e-4, f"{what}: relative error {rel}"
    scale = ((g.double() ** 2).T @ (x.double() ** 2)).sqrt()
    worst = ((dw.double() - ref).abs() / scale.clamp_min(1e-30)).max().item()
    assert worst < 1e-3, f"{what}: worst element error {worst} of sqrt(sum g^2 x^2)"


@pytest.mark.parametrize("cfg,T,n,m", LINEARS, ids=[c[0] for c in LINEARS])
def test_switchback_linear_all_rows(cfg, T, n, m):
    x, w, g = _inputs(T, n, m, seed=[c[0] for c in LINEARS].index(cfg) + 11)
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    ctx = L.LinearContext()
    y = L.linear_forward(mode, x, w, ctx)
    # the layer's own quantized operands, read back from its workspace (sb_linear_workspace_layout)
    v = L.workspace_views(ctx)
    xq_l, xs_l = v["x"].payload.clone(), v["x"].state.clone()
    wq_l, wqt_l, ws_l = v["w"].payload.clone(), v["w_t"].payload.clone(), v["w"].state.clone()
    dx, dw = L.linear_backward(mode, ctx, g)
    gq_l, gs_l = v["g"].payload, v["g"].state
    torch.cuda.synchronize()

    xh, wh, gh = _host_f32(x), _host_f32(w), _host_f32(g)
    xq_o, xs_o = _oracle_q(xh, O.ROW)
    wq_o, ws_o = _oracle_q(wh, O.TENSOR)
    wqt_o, _ = _oracle_q(wh, O.TENSOR_T)
    gq_o, gs_o = _oracle_q(gh, O.ROW)
    del xh, wh, gh

    # payloads and scales the layer wrote: bit-exact on every row
    assert torch.equal(xq_l, xq_o), "X payload differs from the oracle"
    assert torch.equal(xs_l.view(torch.int32), xs_o.view(torch.int32)), "X row states differ"
    assert torch.equal(wq_l, wq_o), "W payload differs from the oracle"
    assert torch.equal(wqt_l, wqt_o), "W^T payload differs from the oracle"
    assert torch.equal(ws_l.view(torch.int32), ws_o.view(torch.int32)), "W tensor state differs"
    assert torch.equal(gq_l, gq_o), "G payload differs from the oracle"
    assert torch.equal(gs_l.view(torch.int32), gs_o.view(torch.int32)), "G row states differ"
    qw_l = L.QuantizedMatrix(wq_l, ws_l, L.TENSOR)
    qg_l = L.QuantizedMatrix(gq_l, gs_l, L.ROW)

    # forward: raw int32 accumulators bit-exact, Y within the bf16 rounding of the formula
    raw = L.int8_matmul_dequant(L.QuantizedMatrix(xq_l, xs_l, L.ROW), qw_l, out_dtype="raw")
    want = _exact_raw(xq_o, wq_o)
    assert torch.equal(raw.double(), want), "forward int32 accumulators differ"
    del raw
    _assert_bf16_close(y, _dequant_ref(want, xs_o, ws_o.expand(m)), "Y")
    del want, y

    # input gradient: dX = deq(qrow(G) qtensor_T(W)) (linear.cpp:234-235)
    qwt = L.QuantizedMatrix(wqt_l, ws_l, L.TENSOR)
    raw = L.int8_matmul_dequant(qg_l, qwt, out_dtype="raw")
    want = _exact_raw(gq_o, wqt_o)
    assert torch.equal(raw.double(), want), "dX int32 accumulators differ"
    del raw
    _assert_bf16_close(dx, _dequant_ref(want, gs_o, ws_o.expand(n)), "dX")
    del want, dx

    # weight gradient: fp32 dW = G^T X over K = T tokens (linear.cpp:245)
    _assert_dw(dw, g, x, "dW")


def test_c1_exact_mode_bit_identical():
    """Config 1 (T=8192, 1024 -> 4096) in exact mode: Y and dX equal the reference's fp64
    epilogue on every element; dW rows equal the reference's sequential fp32 loop
    (matrix.cpp:53-68) computed by the oracle on a row sample (each dW row is independent)."""
    T, n, m = 8192, 1024, 4096
    xh = O.gaussian_matrix(T, n, 0.0, 1.0, O.derive_seed(42, 1))  # bench.cpp:51-53
    wh = O.gaussian_matrix(m, n, 0.0, 1.0, O.derive_seed(42, 2))
    gh = O.gaussian_matrix(T, m, 0.0, 1.0, O.derive_seed(42, 3))
    x, w, g = (torch.from_numpy(a).cuda() for a in (xh, wh, gh))
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8, exact=True)
    ctx = L.LinearContext()
    y = L.linear_forward(mode, x, w, ctx)
    dx, dw = L.linear_backward(mode, ctx, g)
    xq, xs = _oracle_q(xh, O.ROW)
    wq, ws = _oracle_q(wh, O.TENSOR)
    wqt, _ = _oracle_q(wh, O.TENSOR_T)
    gq, gs = _oracle_q(gh, O.ROW)
    assert torch.equal(y, _dequant_ref(_exact_raw(xq, wq), xs, ws.expand(m))), "exact Y"
    assert torch.equal(dx, _dequant_ref(_exact_raw(gq, wqt), gs, ws.expand(n))), "exact dX"
    rows = np.array([0, 1, 777, 2048, 4095])
    dw_o = O.wgrad_f32(np.ascontiguousarray(gh[:, rows]), xh)
    assert np.array_equal(dw[rows].cpu().numpy(), dw_o), "exact dW rows"


def test_c4_switchback_q_and_fp8_payloads_full_size():
    """Config 4 at the ViT-H MLP shape: SwitchBackQ's row-wise W and column-wise (transposed)
    W payloads (linear.cpp:131-132, 226-229) and the fp8 e4m3 / e5m2 row-wise payloads of a
    full T x 5120 operand (quantize.cpp:161-176), all bit-exact against the oracle; the
    SwitchBackQ forward accumulators bit-exact on the full output."""
    T, n, m = T_VIT, 1280, 5120
    x, w, g = _inputs(T, n, m, seed=4)
    wh = _host_f32(w)
    q_row = L.quantize_rowwise(w)
    wq_o, ws_o = _oracle_q(wh, O.ROW)
    assert torch.equal(q_row.payload, wq_o) and torch.equal(q_row.state, ws_o)
    q_colt = L.quantize_columnwise(w, transposed=True)
    wct_o, wcs_o = _oracle_q(np.ascontiguousarray(wh.T), O.ROW)
    assert torch.equal(q_colt.payload, wct_o) and torch.equal(q_colt.state, wcs_o)
    qx = L.quantize_rowwise(x)
    raw = L.matmul_dequant_dual_rowwise(qx, q_row, out_dtype="raw")
    xq_o, _ = _oracle_q(_host_f32(x), O.ROW)
    assert torch.equal(qx.payload, xq_o)
    assert torch.equal(raw.double(), _exact_raw(xq_o, wq_o)), "SwitchBackQ forward accumulators"
    del raw
    gh = _host_f32(g)
    for fmt, ofmt in ((A.SB_E4M3, O.E4M3), (A.SB_E5M2, O.E5M2)):
        q = L.quantize_fp8(g, fmt, L.ROW)
        p_o, s_o = O.quantize_fp8(gh, ofmt, O.ROW)
        assert np.array_equal(q.state.cpu().numpy(), s_o)
        got = fp8_decode(q.payload.cpu().numpy(), fmt)
        assert np.array_equal(got, p_o), f"fp8 fmt {fmt} payload"


def _vit_block_tensors():
    return [(3840, 1280), (1280, 1280), (5120, 1280), (1280, 5120)]  # qkv, out, fc1, fc2


@pytest.mark.parametrize("clipping", [A.SB_CLIP_NONE, A.SB_CLIP_UPDATE])
def test_c5_stableadamw_full_vit_block_bitwise(clipping):
    """Config 5's update rule on a full ViT-H block tensor set (4 tensors, 19.66 M params),
    paper hyper-parameters (beta1 0.9, beta2 0.99, eps 1e-6, lambda 0.2): theta, v and u are
    bit-identical to the oracle after 4 steps. Under update clipping eta = alpha / max(1, RMS)
    is reduction-independent while RMS <= 1: the state starts from a large u and
    the gradients shrink, so RMS < 1 at every step (asserted)."""
    rng = np.random.default_rng(5)
    shapes = _vit_block_tensors()
    th = [rng.standard_normal(r * c).astype(np.float32) * 0.02 for r, c in shapes]
    v = [rng.standard_normal(r * c).astype(np.float32) * 1e-3 for r, c in shapes]
    u = [np.abs(rng.standard_normal(r * c)).astype(np.float32) * 1e-4 + 1e-4 for r, c in shapes]
    pd, vd, ud = ([torch.from_numpy(a.copy()).cuda() for a in arrs] for arrs in (th, v, u))
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3 * t, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.2,
                                clipping=clipping)
    for t in range(3, 7):
        gs = [rng.standard_normal(a.size).astype(np.float32) * np.float32(4e-3 * 0.7 ** t) for a in th]
        rms_o, eta_o = O.stableadamw_step(th, gs, v, u, t, alpha=1e-3 * t, beta1=0.9, beta2=0.99, eps=1e-6,
                                          weight_decay=0.2, clipping=clipping)
        info = L.optimizer_step([L.TensorRef(f"t{i}", p, torch.from_numpy(gi).cuda(), vv, uu)
                                 for i, (p, gi, vv, uu) in enumerate(zip(pd, gs, vd, ud))], hp, t)
        assert (rms_o < 1.0).all()
        np.testing.assert_allclose([r for r, _ in info], rms_o, rtol=1e-12)
        assert [e for _, e in info] == list(eta_o)
    for name, dv, hv in (("theta", pd, th), ("v", vd, v), ("u", ud, u)):
        for i, (a, b) in enumerate(zip(dv, hv)):
            assert np.array_equal(a.cpu().numpy(), b), f"{name}[{i}] differs from the oracle"
