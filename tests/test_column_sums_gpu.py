"""GPU: sb_column_sums, the nn module's bias gradient (sum over tokens of G) — against an fp64
torch sum, deterministic, strided rows, ragged widths, empty input, graph capture."""
import pytest
import torch

from paper_2304_13013_b200 import lowprec as L

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("rows,cols", [(1, 8), (7, 3), (300, 1280), (1000, 3840), (65792, 1280), (4097, 100),
                                       (65792, 5120), (33, 4104)])
def test_matches_fp64_sum(dtype, rows, cols):
    g = torch.Generator(device="cuda").manual_seed(rows * 7 + cols)
    x = torch.randn(rows, cols, device="cuda", generator=g).to(dtype)
    got = L.column_sums(x)
    ref = x.double().sum(0)
    tol = 1e-5 * (rows ** 0.5) * x.double().abs().amax(0).clamp_min(1) + 1e-6
    assert got.dtype == torch.float32 and got.shape == (cols,)
    assert ((got.double() - ref).abs() <= tol).all()
    assert torch.equal(got, L.column_sums(x)), "deterministic"


def test_strided_rows_and_column_slices():
    x = torch.randn(2000, 3840, device="cuda").bfloat16()
    for i in range(3):
        v = x[:, i * 1280:(i + 1) * 1280]  # row stride 3840 > width 1280
        assert torch.equal(L.column_sums(v), L.column_sums(v.contiguous()))
    assert torch.equal(L.column_sums(x.view(20, 100, 3840)), L.column_sums(x))


def test_empty_rows_give_zeros():
    x = torch.empty(0, 64, device="cuda", dtype=torch.bfloat16)
    assert torch.equal(L.column_sums(x), torch.zeros(64, device="cuda"))


def test_graph_capture_replays():
    x = torch.randn(65792, 1280, device="cuda").bfloat16()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        first = L.column_sums(x)  # grows this stream's scratch before the capture
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            out = L.column_sums(x)
    gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, first)
