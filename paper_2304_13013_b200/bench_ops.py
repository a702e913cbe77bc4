"""The reference's op micro-benchmark (``lowprec bench``, proj/core/src/bench.cpp:45-92 and
proj/tools/main.cpp:46-53) on the B200 kernels: same ops, same CSV schema, same size syntax
and errors, timed with CUDA events on the handle's stream instead of steady_clock.

    python -m paper_2304_13013_b200.bench_ops --sizes 8192x1024,65792x1280 --repeats 20 --out ops.csv

Per size ``<b>x<dim>``: X [b x dim], W [dim x dim], G [b x dim], N(0, 1) fp32 on three
seeded streams (bench.cpp:51-53 uses derive_seed(seed, 1|2|3); the timings do not depend on the
values), then the rows quantize_rowwise, quantize_tensorwise, quantize_tensorwise_transpose,
int8_matmul_dequant, matmul, switchback_fwd_bwd and quantize_fraction (bench.cpp:63-89:
(2 q_row + q_tensor + q_tt) / switchback_fwd_bwd). ``matmul`` is the fp32 reference-order
product (sequential, exact); ``switchback_fwd_bwd`` is linear_forward + linear_backward in
SwitchBack int8 with fp32 I/O (the performance path, bf16 is a separate dtype choice).
"""
from __future__ import annotations

import argparse
import re
import sys
from dataclasses import dataclass

import torch

from . import _capi as A
from . import lowprec as L


@dataclass
class BenchRow:  # bench.hpp: op, b, dim, repeats, mean_ns, p50_ns
    op: str
    b: int
    dim: int
    repeats: int
    mean_ns: float
    p50_ns: float


def parse_bench_sizes(text: str) -> list[tuple[int, int]]:
    """bench.cpp:105-124: comma-separated <b>x<dim>, both >= 1."""
    sizes = []
    for tok in text.split(","):
        if not tok:
            continue
        x = tok.find("x")
        if x <= 0 or x + 1 >= len(tok) or not re.fullmatch(r"[+-]?\d+", tok[:x]) or not re.fullmatch(r"[+-]?\d+", tok[x + 1:]):
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT,
                                    f"bench: size token must be <b>x<dim>, got '{tok}'")
        sizes.append((int(tok[:x]), int(tok[x + 1:])))
    if not sizes:
        raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "bench: no sizes given")
    return sizes


def _time_op(repeats: int, op) -> tuple[float, float]:
    """bench.cpp:23-40: one warm-up call, then `repeats` timed calls; (mean_ns, p50_ns)."""
    op()
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(repeats)]
    for a, b in evs:
        a.record(stream)
        op()
        b.record(stream)
    torch.cuda.synchronize()
    ns = sorted(a.elapsed_time(b) * 1e6 for a, b in evs)
    n = len(ns)
    p50 = ns[n // 2] if n % 2 else 0.5 * (ns[n // 2 - 1] + ns[n // 2])
    return sum(ns) / n, p50


def _gaussian(rows: int, cols: int, seed: int, stream: int) -> torch.Tensor:
    """N(0, 1) fp32 on the device. The reference draws from its own Rng streams; the op timings
    do not depend on the values, so a seeded torch generator stands in."""
    g = torch.Generator(device="cuda").manual_seed((seed * 1000003 + stream) & 0x7FFFFFFF)
    return torch.randn(rows, cols, device="cuda", generator=g)


def run_bench(sizes: list[tuple[int, int]], repeats: int, seed: int = 42) -> list[BenchRow]:
    if repeats < 1:
        raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "bench: repeats must be >= 1")
    if not sizes:
        raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "bench: at least one size required")
    h = A.handle()
    h.bind_stream(torch.cuda.current_stream().cuda_stream)
    rows = []
    for b, dim in sizes:
        if b < 1 or dim < 1:
            raise L.InvalidArgument(A.SB_ERR_INVALID_ARGUMENT, "bench: sizes must be >= 1")
        x, w, g = _gaussian(b, dim, seed, 1), _gaussian(dim, dim, seed, 2), _gaussian(b, dim, seed, 3)
        qx = L.quantize_rowwise(x)
        qw = L.quantize_tensorwise(w)
        mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
        ws = L._workspace(mode, b, dim, dim, x.device)
        stats = {}
        stats["quantize_rowwise"] = _time_op(repeats, lambda: L.quantize_rowwise(x, check=False))
        stats["quantize_tensorwise"] = _time_op(repeats, lambda: L.quantize_tensorwise(w, check=False))
        stats["quantize_tensorwise_transpose"] = _time_op(repeats, lambda: L.quantize_tensorwise_transpose(w, check=False))
        stats["int8_matmul_dequant"] = _time_op(repeats, lambda: L.int8_matmul_dequant(qx, qw, exact=False))
        stats["matmul"] = _time_op(repeats, lambda: L.matmul(x, w))

        def sb():
            ctx = L.LinearContext()
            L.linear_forward(mode, x, w, ctx, workspace=ws, check=False)
            L.linear_backward(mode, ctx, g, check=False)

        stats["switchback_fwd_bwd"] = _time_op(repeats, sb)
        for op, (mean, p50) in stats.items():
            rows.append(BenchRow(op, b, dim, repeats, mean, p50))
        # one forward+backward quantizes X and G row-wise and W both tensor-wise ways (bench.cpp:83-89)
        qr, qt, qtt, s = (stats[k] for k in ("quantize_rowwise", "quantize_tensorwise",
                                            "quantize_tensorwise_transpose", "switchback_fwd_bwd"))
        rows.append(BenchRow("quantize_fraction", b, dim, repeats, (2 * qr[0] + qt[0] + qtt[0]) / s[0],
                             (2 * qr[1] + qt[1] + qtt[1]) / s[1]))
    L.check_error()
    return rows


def bench_csv(rows: list[BenchRow]) -> str:
    """bench.cpp:95-103 (15 significant digits)."""
    out = ["op,b,dim,repeats,mean_ns,p50_ns"]
    for r in rows:
        out.append(f"{r.op},{r.b},{r.dim},{r.repeats},{r.mean_ns:.15g},{r.p50_ns:.15g}")
    return "\n".join(out) + "\n"


def main(argv=None) -> int:
    """proj/tools/main.cpp:46-53, 88-92: --sizes, --repeats and --out are required; the CSV is
    written to --out and echoed on stdout; usage errors exit 1."""
    ap = argparse.ArgumentParser(prog="lowprec bench", description="micro-benchmark the quantized kernels")
    ap.add_argument("--sizes", required=True, help="comma-separated <b>x<dim> pairs, e.g. 64x128,256x256")
    ap.add_argument("--repeats", type=int, required=True, help="timed repetitions per op")
    ap.add_argument("--out", required=True, help="CSV output path")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 1 if e.code else 0
    try:
        csv = bench_csv(run_bench(parse_bench_sizes(a.sizes), a.repeats))
        with open(a.out, "w") as f:
            f.write(csv)
    except (L.InvalidArgument, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    sys.stdout.write(csv)
    return 0


if __name__ == "__main__":
    sys.exit(main())
