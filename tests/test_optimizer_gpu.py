"""GPU parity: multi-tensor StableAdamW (optimizer.cpp:102-172)."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import _capi as A
from paper_2304_13013_b200 import lowprec as L
from tests._util import dev, host

pytestmark = pytest.mark.gpu


def refs(ps, gs, vs, us):
    return [L.TensorRef(f"t{i}", p, g, v, u) for i, (p, g, v, u) in enumerate(zip(ps, gs, vs, us))]


@pytest.mark.parametrize("clipping", [A.SB_CLIP_NONE, A.SB_CLIP_UPDATE, A.SB_CLIP_GRAD])
def test_matches_reference_fixture(golden, clipping):
    d = golden("optimizer.npz")
    sizes = [int(r * c) for r, c in d["shapes"]]
    splits = np.cumsum(sizes)[:-1]
    ps = [dev(a) for a in np.split(d[f"theta0_{clipping}"], splits)]
    vs = [torch.zeros(s, device="cuda") for s in sizes]
    us = [torch.zeros(s, device="cuda") for s in sizes]
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 0.01, weight_decay=0.1, clipping=clipping, max_grad_norm=1.0)
    for t in range(1, d[f"grads_{clipping}"].shape[0] + 1):
        gs = [dev(a) for a in np.split(d[f"grads_{clipping}"][t - 1], splits)]
        info = L.optimizer_step(refs(ps, gs, vs, us), hp, t)
        rms = np.array([r for r, _ in info])
        eta = np.array([e for _, e in info])
        np.testing.assert_allclose(rms, d[f"rms_{clipping}"][t - 1], rtol=1e-12)
        np.testing.assert_allclose(eta, d[f"eta_{clipping}"][t - 1], rtol=1e-12)
    th = np.concatenate([host(p) for p in ps])
    if clipping == A.SB_CLIP_NONE:  # no reduction feeds the element math: bitwise
        assert np.array_equal(th, d[f"theta_{clipping}"])
        assert np.array_equal(np.concatenate([host(v) for v in vs]), d[f"v_{clipping}"])
        assert np.array_equal(np.concatenate([host(u) for u in us]), d[f"u_{clipping}"])
    else:
        np.testing.assert_allclose(th, d[f"theta_{clipping}"], rtol=1e-6, atol=1e-7)


def test_bitwise_vs_oracle_50_steps_multi_tensor():  # optimizer_test.cpp:183-205 at scale
    sizes = [4 * 6, 9, 1 << 20, 3 * 4096 + 17]
    rng = np.random.default_rng(0)
    th = [rng.standard_normal(s).astype(np.float32) for s in sizes]
    v = [np.zeros(s, np.float32) for s in sizes]
    u = [np.zeros(s, np.float32) for s in sizes]
    pd, vd, ud = [dev(a) for a in th], [dev(a) for a in v], [dev(a) for a in u]
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 0.003)
    for t in range(1, 51):
        gs = [rng.standard_normal(s).astype(np.float32) * 0.3 for s in sizes]
        O.stableadamw_step(th, gs, v, u, t, alpha=0.003)
        L.optimizer_step(refs(pd, [dev(g) for g in gs], vd, ud), hp, t, infos=False)
    for a, b in zip(pd, th):
        assert np.array_equal(host(a), b)
    for a, b in zip(ud, u):
        assert np.array_equal(host(a), b)


def test_first_step_and_errors():  # optimizer_test.cpp:126-141, :288-303
    p, g = dev([5.0]), dev([3.0])
    v, u = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 0.1)
    info = L.optimizer_step([L.TensorRef("w", p, g, v, u)], hp, 1)
    assert host(v)[0] == 3.0 and host(u)[0] == 9.0 and info[0] == (1.0, 0.1)
    assert host(p)[0] == np.float32(5.0 - 0.1 * (3.0 / (3.0 + 1e-6)))
    with pytest.raises(L.InvalidArgument, match="t must be >= 1"):
        L.optimizer_step([L.TensorRef("w", p, g, v, u)], hp, 0)
    with pytest.raises(L.InvalidArgument, match="lr_schedule not set"):
        L.optimizer_step([L.TensorRef("w", p, g, v, u)], L.OptimizerHyperparams(), 1)
    with pytest.raises(L.InvalidArgument, match="shape mismatch"):
        L.optimizer_step([L.TensorRef("w", p, dev([1.0, 2.0]), v, u)], hp, 1)


def test_update_clip_shrinks_eta():  # optimizer_test.cpp:143-159
    p, v, u = torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda"), torch.zeros(1, device="cuda")
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 0.1, clipping=A.SB_CLIP_UPDATE)
    i1 = L.optimizer_step([L.TensorRef("w", p, dev([100.0]), v, u)], hp, 1)
    assert i1[0][1] == 0.1
    i2 = L.optimizer_step([L.TensorRef("w", p, dev([1000.0]), v, u)], hp, 2)
    assert i2[0][0] > 1.0 and i2[0][1] == pytest.approx(0.1 / i2[0][0], rel=1e-15) and i2[0][1] < 0.1


def test_empty_tensor_reports_nan_rms_and_alpha():  # optimizer.cpp:148-160 with n = 0
    p, g = dev([1.0, 2.0, 3.0, 4.0]), dev([0.5, -0.5, 0.25, 1.0])
    v, u = torch.zeros(4, device="cuda"), torch.zeros(4, device="cuda")
    e = [torch.zeros(0, device="cuda") for _ in range(4)]
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 0.05, clipping=A.SB_CLIP_UPDATE)
    info = L.optimizer_step([L.TensorRef("e", *e), L.TensorRef("w", p, g, v, u)], hp, 1)
    assert np.isnan(info[0][0]) and info[0][1] == 0.05
    assert info[1][1] == 0.05


def _trainer_reference(th, gs, v, u, t, hp_kw, scale, per_tensor_skip):
    """trainer.cpp:127-155 restated over the oracle: filter_nonfinite (optimizer.cpp:83-100),
    grad_absmax of the unscaled gradients, optimizer_step over the tensors that are applied."""
    gf = [(g.astype(np.float64) / scale).astype(np.float32) for g in gs]
    skipped = [not np.isfinite(g).all() for g in gf]
    if not per_tensor_skip and any(skipped):
        skipped = [True] * len(gf)
    absmax = [float(np.max(np.where(np.isnan(g), 0, np.abs(g)), initial=0.0)) for g in gf]
    keep = [i for i in range(len(gf)) if not skipped[i]]
    rms = [np.nan] * len(gf)
    if keep:
        r, _ = O.stableadamw_step([th[i] for i in keep], [gf[i] for i in keep], [v[i] for i in keep],
                                  [u[i] for i in keep], t, **hp_kw)
        for j, i in enumerate(keep):
            rms[i] = r[j]
    return skipped, absmax, rms


@pytest.mark.parametrize("scale", [1.0, 1024.0, 3.0])
@pytest.mark.parametrize("per_tensor_skip", [True, False])
@pytest.mark.parametrize("clipping", [A.SB_CLIP_NONE, A.SB_CLIP_GRAD])
def test_fused_trainer_update_matches_reference(scale, per_tensor_skip, clipping):
    """sb_stableadamw_step_ex: unscale + per-tensor skip + grad_absmax + the in-step clip over the
    applied tensors, fused into the optimizer's passes, against the reference trainer path. A
    tensor with an inf gradient is skipped (state untouched, rms = NaN), or the whole step is."""
    rng = np.random.default_rng(int(scale) + 7 * per_tensor_skip + clipping)
    sizes = [3000, 1 << 16, 4096 + 3, 12288]
    th = [rng.standard_normal(s).astype(np.float32) for s in sizes]
    v = [(rng.standard_normal(s) * 1e-3).astype(np.float32) for s in sizes]
    u = [(np.abs(rng.standard_normal(s)) * 1e-4).astype(np.float32) for s in sizes]
    gs = [(rng.standard_normal(s) * 0.05 * scale).astype(np.float32) for s in sizes]
    gs[2][17] = np.inf
    gs[1][5] = np.nan
    gs[1][5] = 0.25  # tensor 1 stays finite; NaN never wins grad_absmax
    hp_kw = dict(alpha=3e-3, weight_decay=0.1, clipping=clipping, max_grad_norm=0.5)
    pd, vd, ud = ([torch.from_numpy(a.copy()).cuda() for a in arrs] for arrs in (th, v, u))
    gd = [torch.from_numpy(g.copy()).cuda() for g in gs]
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 3e-3, weight_decay=0.1, clipping=clipping, max_grad_norm=0.5)
    out = L.optimizer_step_ex(refs(pd, gd, vd, ud), hp, 2, L.LossScaler(scale, per_tensor_skip))
    skipped, absmax, rms = _trainer_reference(th, gs, v, u, 2, hp_kw, scale, per_tensor_skip)
    assert out["skipped"].cpu().tolist() == [int(s) for s in skipped]
    assert out["grad_absmax"].cpu().tolist() == pytest.approx(absmax, rel=0, abs=0)
    got_rms = out["rms"].cpu().numpy()
    np.testing.assert_allclose(got_rms, rms, rtol=1e-12)  # NaN == NaN for skipped tensors
    for name, dv, hv in (("theta", pd, th), ("v", vd, v), ("u", ud, u)):
        for i, (a, b) in enumerate(zip(dv, hv)):
            if clipping == A.SB_CLIP_NONE:
                assert np.array_equal(a.cpu().numpy(), b), f"{name}[{i}]"
            else:  # the global norm's sum order differs, and the clip factor scales g: within rounding
                np.testing.assert_allclose(a.cpu().numpy(), b, rtol=1e-6, atol=1e-7)


def test_shadow_weight_and_absmax_feed_the_next_forward():
    """The theta update writes bf16(theta') and its tensor-wise absmax (optimizer.cpp:162-167 ->
    quantize.cpp:139-141): the shadow equals theta.to(bf16), the word its max |.|, and quantizing
    the shadow with the word gives the payload / state of quantize_tensorwise bit for bit; the
    layer forward that takes the word (sb_linear_forward_ex) equals the plain one."""
    torch.manual_seed(0)
    m, n = 1280, 640
    p = torch.randn(m, n, device="cuda") * 0.02
    g, v, u = torch.randn(m, n, device="cuda") * 1e-3, torch.zeros(m, n, device="cuda"), torch.zeros(m, n, device="cuda")
    shadow = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    word = torch.full((1,), 12345, device="cuda", dtype=torch.int32)  # stale value: the step resets it
    hp = L.OptimizerHyperparams(lr_schedule=lambda t: 1e-3, weight_decay=0.2, clipping=A.SB_CLIP_UPDATE)
    L.optimizer_step_ex([L.TensorRef("w", p, g, v, u)], hp, 1, shadows=[(shadow, word)])
    ref = p.to(torch.bfloat16)
    assert torch.equal(shadow, ref)
    assert word.item() == (ref.view(torch.int16).int() & 0x7FFF).max().item() << 16
    q0, qt0 = L.quantize_tensorwise(ref, with_transpose=True)
    q1, qt1 = L.quantize_tensorwise_from_absmax(shadow, word, with_transpose=True)
    assert torch.equal(q0.payload, q1.payload) and torch.equal(qt0.payload, qt1.payload)
    assert torch.equal(q0.state, q1.state)
    x = torch.randn(4096, n, device="cuda").bfloat16()
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    bias = torch.randn(m, device="cuda")
    c0, c1 = L.LinearContext(), L.LinearContext()
    y0 = L.linear_forward(mode, x, shadow, c0, bias=bias)
    y1 = L.linear_forward(mode, x, shadow, c1, bias=bias, w_absmax=word)
    assert torch.equal(y0, y1)
    gy = torch.randn(4096, m, device="cuda").bfloat16()
    assert all(torch.equal(a, b) for a, b in zip(L.linear_backward(mode, c0, gy), L.linear_backward(mode, c1, gy)))
