"""SwitchBack fwd+bwd throughput (BASELINE.json metric) on B200.

Default workload = config 2 (BASELINE.json configs[1]): the CLIP ViT-Huge MLP block,
fc1 1280->5120 and fc2 5120->1280, 256 images x 257 tokens = 65792 tokens per GPU,
SwitchBack int8 (row-wise X/G, tensor-wise W) forward + input gradient on tcgen05
kind::i8, bf16 weight gradient on tcgen05 kind::f16. One step = forward + backward of
both linears (the reference's switchback_fwd_bwd unit, bench.cpp:75-81), each with its
own synthetic bf16 input and output gradient. N > 1: weak scaling, each rank owns 65792
tokens; dW all-reduce (NCCL) is the only collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

T_PER_GPU = 256 * 257
LAYERS = [("fc1", 1280, 5120), ("fc2", 5120, 1280)]  # (name, n = in_features, m = out_features)
METRIC = "SwitchBack fwd+bwd tokens/s at ViT-H shapes (1/2/4/8 GPU); int8 TOPS % of peak"
WORKLOAD = "CLIP ViT-Huge MLP block 1280->5120->1280, 256 images x 257 tokens, int8 fwd/dX + bf16 dW"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
                f = [s.strip() for s in out.strip().split(",")]
                if len(f) == 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU side
def cpu_reference_rate(budget_s: float = 12.0, threads: int | None = None):
    """The UNMODIFIED reference (oracle/_ref: lowprec::linear_forward + linear_backward,
    {kSwitchBack, kInt8}) on all host threads over a bounded token sample of both C2
    linears. Returns (tokens/s, cores, sample description, kind)."""
    import numpy as np

    import oracle as O

    threads = threads or os.cpu_count() or 1
    kind = "reference" if O.ref_available() else "port"
    rows = max(threads, 8)
    # calibrate: grow the per-layer token sample until one pass takes >= budget/4
    total_t = 0.0
    total_tok = 0
    while True:
        t0 = time.perf_counter()
        for _, n, m in LAYERS:
            x = np.random.default_rng(1).standard_normal((rows, n)).astype(np.float32)
            w = (np.random.default_rng(2).standard_normal((m, n)) / np.sqrt(n)).astype(np.float32)
            g = np.random.default_rng(3).standard_normal((rows, m)).astype(np.float32)
            if kind == "reference":
                rc = O.ref().ref_switchback_fwd_bwd_threaded(x, w, g, rows, n, m, threads, None, None, None)
                assert rc == 0
            else:
                O.switchback_forward(x, w)
                O.switchback_backward(x, w, g)
        dt = time.perf_counter() - t0
        total_t += dt
        total_tok += rows
        if total_t >= budget_s or dt >= budget_s / 3:
            break
        rows = int(rows * max(2.0, min(8.0, (budget_s / 3) / max(dt, 1e-3))))
    sample = (f"{total_tok} tokens through fc1+fc2 (1280->5120, 5120->1280) SwitchBack int8 fwd+bwd, "
              f"token rows sharded over {threads if kind == 'reference' else 1} threads; cost is linear in tokens")
    return total_tok / total_t, threads if kind == "reference" else 1, sample, kind


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rates = []
    for _ in range(args.warmup):
        pass
    for _ in range(max(1, args.steps)):
        r, cores, sample, kind = cpu_reference_rate(budget_s=args.ref_budget)
        rates.append(r)
    v = sum(rates) / len(rates)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T_PER_GPU / v * 1000.0, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8+f32 (reference CPU)", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD + " (CPU reference, bounded token sample)", "tokens_per_gpu": T_PER_GPU},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side
def run_ours(args):
    import torch

    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200 import dp
    from paper_2304_13013_b200 import lowprec as L

    rank, world, local = dp.init_from_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    T = args.tokens
    mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8)
    cmode = mode.c()
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)

    def randn(*shape, scale=1.0):
        return (torch.randn(*shape, device=dev, generator=gen) * scale).to(torch.bfloat16)

    layers = []
    for name, n, m in LAYERS:
        lay = {"name": name, "n": n, "m": m,
               "x": randn(T, n), "w": randn(m, n, scale=n ** -0.5), "g": randn(T, m),
               "y": torch.empty(T, m, device=dev, dtype=torch.bfloat16),
               "dx": torch.empty(T, n, device=dev, dtype=torch.bfloat16),
               "gq": torch.empty(T, m, device=dev, dtype=torch.int8),
               "gs": torch.empty(T, device=dev, dtype=torch.float32),
               "dw": torch.empty(m, n, device=dev, dtype=torch.float32), "ctx": A.LinearCtx()}
        lay["ws"] = L._workspace(mode, T, n, m, dev)
        layers.append(lay)
    h = A.handle(local)
    P = L._p

    # The step's kernels, straight through the C-ABI (the same launches sb_linear_forward /
    # sb_linear_backward issue; the backward is split so the dW GEMM can be timed alone).
    def fwd(lay):
        A.check(h.lib.sb_linear_forward(h.h, C.byref(cmode), P(lay["x"]), P(lay["w"]), A.SB_BF16, T, lay["n"],
                                        lay["m"], P(lay["y"]), C.byref(lay["ctx"]), P(lay["ws"]), lay["ws"].numel()))

    def bwd_dx(lay):
        c = lay["ctx"]
        A.check(h.lib.sb_quantize_rowwise(h.h, P(lay["g"]), A.SB_BF16, T, lay["m"], lay["m"], P(lay["gq"]), lay["m"],
                                          P(lay["gs"])))
        A.check(h.lib.sb_gemm_i8(h.h, P(lay["gq"]), P(lay["gs"]), C.c_void_p(c.w_q_t), C.c_void_p(c.w_state),
                                 A.SB_SCALE_ROW_TENSOR, T, lay["n"], lay["m"], P(lay["dx"]), A.SB_BF16, 0))

    def bwd_dw(lay):
        A.check(h.lib.sb_wgrad(h.h, P(lay["g"]), P(lay["x"]), A.SB_BF16, T, lay["m"], lay["n"], P(lay["dw"]), 0, 0))

    fc1, fc2 = layers
    segments = [lambda: (fwd(fc1), fwd(fc2), bwd_dx(fc2)), lambda: bwd_dw(fc2), lambda: bwd_dx(fc1),
                lambda: bwd_dw(fc1)]
    stream = torch.cuda.current_stream(dev)
    ar = dp.GradAllReduce()

    # warmup (eager), counting launches of one step
    for i in range(max(1, args.warmup)):
        l0 = h.launches()
        h.bind_stream(stream.cuda_stream)
        for seg in segments:
            seg()
        launches_per_step = h.launches() - l0
    torch.cuda.synchronize()
    graphs = None
    if not args.no_graph:
        graphs = []
        for seg in segments:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                h.bind_stream(torch.cuda.current_stream(dev).cuda_stream)
                seg()
            graphs.append(g)
        h.bind_stream(stream.cuda_stream)
        for g in graphs:
            g.replay()
        torch.cuda.synchronize()

    run = [g.replay for g in graphs] if graphs else segments
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]

    def step(e):
        run[0]()
        e[0].record(stream)
        run[1]()          # dW fc2
        e[1].record(stream)
        ar.launch(fc2["dw"])
        run[2]()
        e[2].record(stream)
        run[3]()          # dW fc1
        e[3].record(stream)
        ar.launch(fc1["dw"])
        ar.wait()

    if world > 1:
        torch.distributed.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        start.record(stream)
        for i in range(args.steps):
            step(ev[i])
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end) / args.steps
    ms = dp.max_over_ranks(ms, dev)
    value = T * world / (ms / 1000.0)
    launches = launches_per_step * args.steps

    # dominant kernel: the bf16 dW GEMM (2*m*n*T flops per launch), timed by the events
    # bracketing its graph segment inside the timed region
    dw_times = [e[0].elapsed_time(e[1]) + e[2].elapsed_time(e[3]) for e in ev]
    pk = peaks()
    flops_step = sum(2.0 * lay["m"] * lay["n"] * T for lay in layers)
    achieved = flops_step * args.steps / (sum(dw_times) / 1000.0) / 1e12
    peak = pk["bf16_tflops_sustained"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "dw_gemm_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("bytes_per_launch")
    share = sum(dw_times) / (ms * args.steps)
    int8_ops_step = sum(4.0 * lay["m"] * lay["n"] * T for lay in layers)

    e2e = None
    if rank == 0 and not args.no_e2e:
        e2e = e2e_host(args, L, torch)
    yard = cublas_yardstick(torch, layers, T, args) if rank == 0 else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r, cores, sample, kind = cpu_reference_rate(budget_s=args.ref_budget)
        cpu = {"value": r, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "int8 (fwd, dX) + bf16 (dW), fp32 accumulate", "data": "synthetic",
                "config": {"workload": WORKLOAD, "tokens_per_gpu": T, "global_tokens": T * world,
                           "layers": [f"{n}->{m}" for _, n, m in LAYERS], "parallelism": f"dp{world} (token shards)",
                           "l2": "inputs larger than L2 (X, G, H operands 168-673 MB each)",
                           "cuda_graphs": graphs is not None},
                "gpu_launches": launches,
                "roofline": {"bound": "tensor", "kernel": "bf16 dW GEMM (tcgen05 kind::f16, MN-major)",
                             "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                             "peak_source": f"{pk['source']} bf16 sustained (MEASURED_PEAKS.json)", "traffic": traffic,
                             "share_of_step": share, "flops_per_launch": [2 * lay["m"] * lay["n"] * T for lay in layers]},
                "int8_tops_per_step": int8_ops_step / 1e12,
                "clocks": clk.summary(),
                "e2e": e2e, "cpu_baseline": cpu, "yardstick_cublas_bf16": yard}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_host(args, L, torch):
    """Same workload through the C-ABI host-buffer entry sb_switchback_fwd_bwd_host:
    pinned host X, W, G in; Y, dX, dW out, every step."""
    T = args.tokens
    bufs = []
    g = torch.Generator().manual_seed(7)
    for _, n, m in LAYERS:
        x = torch.randn(T, n, generator=g).to(torch.bfloat16).pin_memory()
        w = (torch.randn(m, n, generator=g) / n ** 0.5).to(torch.bfloat16).pin_memory()
        gg = torch.randn(T, m, generator=g).to(torch.bfloat16).pin_memory()
        bufs.append((x, w, gg))
    h2d = sum(x.numel() * 2 + w.numel() * 2 + gg.numel() * 2 for x, w, gg in bufs)
    d2h = sum(x.shape[0] * w.shape[0] * 2 + x.numel() * 2 + w.numel() * 4 for x, w, gg in bufs)
    for _ in range(max(1, args.warmup // 2)):
        for x, w, gg in bufs:
            L.switchback_fwd_bwd_host(x, w, gg)
    steps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        for x, w, gg in bufs:
            L.switchback_fwd_bwd_host(x, w, gg)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return {"value": T / dt, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "sb_switchback_fwd_bwd_host (C-ABI, pinned host buffers, chunked H2D/compute/D2H overlap)",
            "steps": steps}


def cublas_yardstick(torch, layers, T, args):
    """bf16 Standard linear through cuBLAS (torch.matmul): Y = X W^T, dX = G W, dW = G^T X."""
    def once():
        for lay in layers:
            x, w, g = lay["x"], lay["w"], lay["g"]
            torch.matmul(x, w.t())
            torch.matmul(g, w)
            torch.matmul(g.t(), x)
    for _ in range(2):
        once()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, min(args.steps, 10))
    s.record()
    for _ in range(n):
        once()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / n
    return {"value": T / (ms / 1000.0), "unit": "tokens/s", "ms_per_step": ms}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tokens", type=int, default=T_PER_GPU)
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
