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
