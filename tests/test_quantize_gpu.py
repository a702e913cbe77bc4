"""GPU parity: quantize kernels (K1-K4, K8, K10) vs the oracle — bit-exact."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import lowprec as L
from tests._util import adversarial, bf16, dev, fp8_decode, host

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (3, 5), (13, 70), (7, 8), (64, 1024), (37, 1280), (33, 5120), (9, 8200), (5, 16384), (2, 40000),
          (2000, 5120), (700, 10240), (4000, 1280)]  # many rows per block: ring wrap-around with few stages


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rowwise_bit_exact(shape, dtype):
    x = adversarial(*shape, seed=sum(shape))
    if dtype == torch.bfloat16:
        x = bf16(x)
    q = L.quantize_rowwise(dev(x, dtype))
    qo, so = O.quantize(x, O.ROW)
    assert np.array_equal(host(q.payload), qo)
    assert np.array_equal(host(q.state), so)


@pytest.mark.parametrize("scale", [1e-38, 1e-20, 1.0, 1e20, 5e37])
def test_rowwise_random_scales_fp32(scale):
    rng = np.random.default_rng(1)
    x = (rng.standard_normal((257, 333)) * scale).astype(np.float32)
    q = L.quantize_rowwise(dev(x))
    qo, so = O.quantize(x, O.ROW)
    assert np.array_equal(host(q.payload), qo) and np.array_equal(host(q.state), so)


def test_rowwise_every_tie_exhaustive_bf16():
    # all 2^16 bf16 bit patterns that are finite, against a row state of 2.0 (ties at p/2*2/127)
    u = np.arange(0, 65536, dtype=np.uint32) << 16
    v = u.view(np.float32)
    v = v[np.isfinite(v) & (np.abs(v) <= 2.0)]
    x = np.concatenate([v, [2.0]]).astype(np.float32)
    pad = (-x.size) % 8
    x = np.concatenate([x, np.zeros(pad, np.float32)]).reshape(1, -1)
    q = L.quantize_rowwise(dev(x, torch.bfloat16))
    qo, so = O.quantize(x, O.ROW)
    assert np.array_equal(host(q.payload), qo) and np.array_equal(host(q.state), so)


def _bf16_tie_rows(cols):
    """One row per bf16 state mantissa (128 rows, state 1.xxx * 2^3): the row holds the state and
    every bf16 magnitude in [state * 2^-9, state] of both signs (all inputs with a nonzero payload,
    every exact half-integer tie 127|x|/s = k + 1/2 among them), then random fill <= state."""
    rng = np.random.default_rng(0)
    rows = []
    for b in range(128, 256):
        st = np.float32(b / 128.0 * 8.0)
        u = np.arange(0, 1 << 15, dtype=np.uint32) << 16
        v = u.view(np.float32)
        v = v[(v <= st) & (v >= st * 2.0 ** -9)]
        row = np.concatenate([[st], v, -v]).astype(np.float32)
        assert row.size <= cols
        fill = bf16((rng.uniform(-1, 1, cols - row.size) * st).astype(np.float32))
        rows.append(np.concatenate([row, fill]))
    return np.stack(rows).astype(np.float32)


@pytest.mark.parametrize("cols", [4096, 5120, 6144])
def test_rowwise_bf16_ties_every_state_mantissa(cols):
    """The bf16 one-FMA path (qvec_bf16_fast) against the reference rounding for every state
    mantissa, including 1.984375 (= 254/128, the mantissa with ties at every odd multiple)."""
    x = _bf16_tie_rows(cols)
    q = L.quantize_rowwise(dev(x, torch.bfloat16))
    qo, so = O.quantize(x, O.ROW)
    assert np.array_equal(host(q.state), so)
    assert np.array_equal(host(q.payload), qo)


def test_rowwise_smem_ring_kernel_subprocess():
    """The TMA/smem-ring row kernel (SB_QUANT_KERNEL=tma) on shapes with many rows per block
    and ring wrap-around, including the slot-ownership case (stages not a multiple of warps)."""
    import subprocess
    import sys
    import textwrap

    code = textwrap.dedent("""
        import numpy as np, torch, sys
        sys.path.insert(0, '.')
        import oracle as O
        from paper_2304_13013_b200 import lowprec as L
        from tests._util import adversarial, bf16, dev, host
        for shape in [(4000, 1280), (3000, 1024), (2000, 5120), (700, 10240), (513, 2000)]:
            for dt in (torch.float32, torch.bfloat16):
                x = adversarial(*shape, seed=sum(shape))
                if dt == torch.bfloat16:
                    x = bf16(x)
                q = L.quantize_rowwise(dev(x, dt))
                qo, so = O.quantize(x, O.ROW)
                assert np.array_equal(host(q.payload), qo), (shape, dt)
                assert np.array_equal(host(q.state), so), (shape, dt)
        print("ok")
    """)
    import os

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env={**os.environ, "SB_QUANT_KERNEL": "tma"},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_rowwise_nonfinite_raises():
    x = np.ones((4, 64), np.float32)
    x[2, 5] = np.nan
    with pytest.raises(L.InvalidArgument, match="quantize_rowwise: non-finite input"):
        L.quantize_rowwise(dev(x))
    x[2, 5] = np.inf
    with pytest.raises(L.InvalidArgument, match="non-finite"):
        L.quantize_rowwise(dev(x, torch.bfloat16))
    L.quantize_rowwise(dev(np.ones((4, 64), np.float32)))  # latch cleared


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (13, 70), (64, 64), (130, 70), (1280, 5120), (5120, 1280), (72, 136),
                                   (3840, 1280), (1000, 8), (8, 1000)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_tensorwise_and_transpose_bit_exact(shape, dtype):
    x = adversarial(*shape, seed=3)
    x[4:5] = 0 if shape[0] > 4 else x[4:5]  # keep one global absmax from the "huge" row out of the way
    if dtype == torch.bfloat16:
        x = bf16(x)
    q, qt = L.quantize_tensorwise(dev(x, dtype), with_transpose=True)
    qo, so = O.quantize(x, O.TENSOR)
    qto, sto = O.quantize(x, O.TENSOR_T)
    assert np.array_equal(host(q.payload), qo) and np.array_equal(host(q.state), so)
    assert np.array_equal(host(qt.payload), qto)
    q2 = L.quantize_tensorwise_transpose(dev(x, dtype))
    assert np.array_equal(host(q2.payload), qto) and np.array_equal(host(q2.state), sto)


@pytest.mark.parametrize("b", [128, 160, 201, 254, 255])
def test_tensorwise_bf16_ties(b):
    """Tensor state with mantissa b/128 and every bf16 magnitude below it (all exact ties) —
    the fused one-launch tensor-wise kernel's one-FMA path against the reference rounding."""
    st = np.float32(b / 128.0 * 4.0)
    u = np.arange(0, 1 << 15, dtype=np.uint32) << 16
    v = u.view(np.float32)
    v = v[(v <= st) & (v >= st * 2.0 ** -9)]
    row = np.concatenate([[st], v, -v]).astype(np.float32)
    cols = 64
    row = np.concatenate([row, np.zeros((-row.size) % cols, np.float32)])
    x = row.reshape(-1, cols)
    q, qt = L.quantize_tensorwise(dev(x, torch.bfloat16), with_transpose=True)
    qo, so = O.quantize(x, O.TENSOR)
    assert np.array_equal(host(q.payload), qo) and np.array_equal(host(q.state), so)
    assert np.array_equal(host(qt.payload), qo.T)


def test_tensorwise_nonfinite_raises():
    x = np.ones((256, 512), np.float32)
    x[100, 7] = np.inf
    with pytest.raises(L.InvalidArgument, match="non-finite"):
        L.quantize_tensorwise(dev(x, torch.bfloat16))
    q = L.quantize_tensorwise(dev(np.ones((256, 512), np.float32), torch.bfloat16))  # latch cleared, words reset
    assert host(q.state)[0] == 1.0 and (host(q.payload) == 127).all()


@pytest.mark.parametrize("shape", [(1, 1), (2, 3), (13, 70), (300, 77), (1280, 5120)])
def test_columnwise_bit_exact(shape):
    x = adversarial(*shape, seed=5).T.copy() if shape[0] > 7 else adversarial(*shape, seed=5)
    q = L.quantize_columnwise(dev(x))
    qo, so = O.quantize(x, O.COL)
    assert np.array_equal(host(q.payload), qo) and np.array_equal(host(q.state), so)
    qt = L.quantize_columnwise(dev(x), transposed=True)  # == quantize_rowwise(x^T)
    qro, sro = O.quantize(x.T.copy(), O.ROW)
    assert np.array_equal(host(qt.payload), qro) and np.array_equal(host(qt.state), sro)


@pytest.mark.parametrize("axis", [L.ROW, L.COLUMN, L.TENSOR])
def test_dequantize_bit_exact(axis):
    x = adversarial(29, 77, seed=9)
    ax = {L.ROW: O.ROW, L.COLUMN: O.COL, L.TENSOR: O.TENSOR}[axis]
    qo, so = O.quantize(x, ax)
    q = L.QuantizedMatrix(dev(qo, torch.int8), dev(so), axis)
    assert np.array_equal(host(L.dequantize(q)), O.dequantize(qo, so, ax))


@pytest.mark.parametrize("shape", [(41, 97), (40, 96), (33, 5120), (300, 1280)])  # generic + vectorised kernels
@pytest.mark.parametrize("fmt", [L.E4M3, L.E5M2])
@pytest.mark.parametrize("axis", [L.ROW, L.COLUMN, L.TENSOR])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_fp8_quantize_bit_exact(fmt, axis, dtype, shape):
    x = adversarial(*shape, seed=fmt * 3 + axis)
    x[4] = 0
    if dtype == torch.bfloat16:
        x = bf16(x)
    q = L.quantize_fp8(dev(x, dtype), fmt, axis)
    ofmt = O.E4M3 if fmt == L.E4M3 else O.E5M2
    oax = {L.ROW: O.ROW, L.COLUMN: O.COL, L.TENSOR: O.TENSOR}[axis]
    po, so = O.quantize_fp8(x, ofmt, oax)
    assert np.array_equal(fp8_decode(host(q.payload), fmt), po)
    assert np.array_equal(host(q.state), so)
    y = L.dequantize(q)
    want = (po.astype(np.float64) * (so[:, None] if oax == O.ROW else so[None, :] if oax == O.COL else so[0])).astype(np.float32)
    assert np.array_equal(host(y), want)


def test_golden_fixture_quantize(golden):
    d = golden("quantize.npz")
    for key, prefix in (("x_adv", ""), ("x_g", "g_")):
        x = d[key]
        assert np.array_equal(host(L.quantize_rowwise(dev(x)).payload), d[prefix + "q_row"])
        assert np.array_equal(host(L.quantize_columnwise(dev(x)).payload), d[prefix + "q_col"])
        assert np.array_equal(host(L.quantize_tensorwise(dev(x)).payload), d[prefix + "q_tensor"])
        assert np.array_equal(host(L.quantize_tensorwise_transpose(dev(x)).payload), d[prefix + "q_tensor_t"])
        p = L.quantize_fp8(dev(x), L.E4M3, L.ROW)
        assert np.array_equal(fp8_decode(host(p.payload), 0), d[prefix + "fp8_e4m3_row"])


def test_standalone_quantizers_capture_in_cuda_graph():
    """The ops that use the handle's scratch words (tensor-wise, column-wise) can be captured in a
    CUDA graph on a stream the handle has never run on (no allocation while capturing), and the
    replay equals the eager result."""
    torch.manual_seed(5)
    x = torch.randn(1024, 768, device="cuda").to(torch.bfloat16)
    t_ref = L.quantize_tensorwise(x)
    c_ref = L.quantize_columnwise(x)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            t = L.quantize_tensorwise(x, check=False)
            c = L.quantize_columnwise(x, check=False)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(t.payload, t_ref.payload) and torch.equal(t.state, t_ref.state)
    assert torch.equal(c.payload, c_ref.payload) and torch.equal(c.state, c_ref.state)
