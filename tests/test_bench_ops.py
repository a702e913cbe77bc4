"""The reference's `lowprec bench` op table (bench.cpp:45-124, tools/main.cpp:46-53,
cli_test.cpp:157-188) on the B200 kernels: size parsing and usage errors on CPU, the CSV
schema on the GPU."""
import os

import pytest

from paper_2304_13013_b200 import bench_ops as B
from paper_2304_13013_b200 import lowprec as L


def test_parse_bench_sizes():
    assert B.parse_bench_sizes("4x8,2x16") == [(4, 8), (2, 16)]
    for bad in ("4y8", "x8", "4x", "4x8x2"):
        with pytest.raises(L.InvalidArgument, match="size token must be <b>x<dim>"):
            B.parse_bench_sizes(bad)
    with pytest.raises(L.InvalidArgument, match="no sizes given"):
        B.parse_bench_sizes(",")


def test_usage_errors_exit_one(tmp_path):  # cli_test.cpp:181-188
    assert B.main(["--sizes", "4x8"]) == 1  # --repeats / --out missing
    assert B.main(["--sizes", "4y8", "--repeats", "1", "--out", os.devnull]) == 1


@pytest.mark.gpu
def test_bench_writes_the_csv_schema(tmp_path, capsys):  # cli_test.cpp:157-171
    out = tmp_path / "bench.csv"
    assert B.main(["--sizes", "4x8,2x16", "--repeats", "3", "--out", str(out)]) == 0
    csv = out.read_text()
    assert capsys.readouterr().out == csv  # echoed verbatim
    assert csv.startswith("op,b,dim,repeats,mean_ns,p50_ns\n")
    assert "quantize_rowwise,4,8,3," in csv and "switchback_fwd_bwd,2,16,3," in csv and "quantize_fraction" in csv
    assert csv.count("\n") == 1 + 2 * 7


@pytest.mark.gpu
def test_bench_vit_h_shape_quantize_fraction():
    """The paper's claim: quantize ops take <= 25% of the SwitchBack layer's
    time, ~10% or less at large dim. At the ViT-H width on the B200 kernels."""
    rows = {r.op: r for r in B.run_bench([(65792, 1280)], 5)}
    assert 0 < rows["quantize_fraction"].mean_ns < 0.25
