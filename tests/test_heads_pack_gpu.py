"""GPU parity of sb_heads_pack_quantize (the attention-gradient producer fusion, SURVEY.md §8f row
1): three head-major gradients dq, dk, dv [B, H, S, Dh] -> the packed q/k/v output gradient
G [B*S, 3*H*Dh] (a pure layout move: bit-identical to torch's permute + reshape) and each
projection's row-wise int8 payload / states, bit-identical to the C oracle's quantize_rowwise
(quantize.cpp:116-133) of G's column block — over adversarial rows (zeros, ties, subnormal and
huge scales), strided (non-contiguous) sources, ragged head counts, and non-finite input."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2304_13013_b200 import lowprec as L
from tests._util import adversarial, bf16, host

pytestmark = pytest.mark.gpu


def _heads(B, H, S, Dh, seed, layout="bhsd"):
    """Three bf16 gradients [B, H, S, Dh] holding adversarial rows, in the given memory layout
    (bhsd: contiguous; bshd: the [B, S, H, Dh] buffer attention kernels often write, viewed as
    [B, H, S, Dh])."""
    out = []
    for i in range(3):
        rows = bf16(adversarial(B * S, H * Dh, seed=seed + i))  # row t = b S + s, column h Dh + d
        t = torch.from_numpy(rows).to("cuda", torch.bfloat16).view(B, S, H, Dh)
        out.append(t.permute(0, 2, 1, 3) if layout == "bshd" else t.permute(0, 2, 1, 3).contiguous())
    return out


def _packed_reference(ts):
    B, H, S, Dh = ts[0].shape
    return torch.cat([t.permute(0, 2, 1, 3).reshape(B * S, H * Dh) for t in ts], dim=1)


@pytest.mark.parametrize("B,H,S,Dh", [(2, 16, 257, 80), (1, 1, 7, 8), (3, 5, 33, 24), (1, 8, 100, 64),
                                      (2, 16, 64, 128)])
@pytest.mark.parametrize("layout", ["bhsd", "bshd"])
def test_pack_and_payload_bit_exact(B, H, S, Dh, layout):
    ts = _heads(B, H, S, Dh, seed=B * 1000 + H * 10 + S, layout=layout)
    g, qs = L.heads_pack_quantize(*ts, check=False)
    ref = _packed_reference(ts)
    assert torch.equal(g, ref), "packed G"
    D = H * Dh
    gh = host(g.float())
    for i, q in enumerate(qs):
        qo, so = O.quantize(np.ascontiguousarray(gh[:, i * D:(i + 1) * D]), O.ROW)
        assert np.array_equal(host(q.payload), qo), f"payload {i}"
        assert np.array_equal(host(q.state), so), f"states {i}"
        qr = L.quantize_rowwise(ref[:, i * D:(i + 1) * D].contiguous(), check=False)
        assert torch.equal(q.payload, qr.payload) and torch.equal(q.state, qr.state)


def test_vit_h_shape_full_size():
    """The ViT-H attention shape (256 x 257 tokens, 16 heads x 80): G and all three payloads equal
    the torch packing + the standalone quantizer on every row."""
    B, H, S, Dh = 256, 16, 257, 80
    gen = torch.Generator(device="cuda").manual_seed(5)
    ts = [torch.randn(B, S, H, Dh, device="cuda", generator=gen).bfloat16().permute(0, 2, 1, 3) for _ in range(3)]
    g, qs = L.heads_pack_quantize(*ts)
    ref = _packed_reference(ts)
    assert torch.equal(g, ref)
    D = H * Dh
    for i, q in enumerate(qs):
        qr = L.quantize_rowwise(ref[:, i * D:(i + 1) * D].contiguous())
        assert torch.equal(q.payload, qr.payload) and torch.equal(q.state, qr.state)


def test_nonfinite_raises_and_clears():
    ts = _heads(1, 2, 9, 16, seed=3)
    ts[1][0, 1, 4, 3] = float("nan")
    with pytest.raises(L.InvalidArgument, match="non-finite"):
        L.heads_pack_quantize(*ts)
    ts[1][0, 1, 4, 3] = 0.0
    L.heads_pack_quantize(*ts)  # latch cleared


def test_argument_errors():
    ts = _heads(1, 2, 9, 16, seed=4)
    with pytest.raises(L.InvalidArgument):
        L.heads_pack_quantize(ts[0], ts[1][:, :, :8], ts[2])
    with pytest.raises(L.InvalidArgument):
        L.heads_pack_quantize(ts[0].float(), ts[1], ts[2])
    big = torch.zeros(1, 32, 4, 72, device="cuda", dtype=torch.bfloat16)  # H * Dh = 2304 > 2048
    with pytest.raises(L.SBError):
        L.heads_pack_quantize(big, big, big)
