"""SwitchBack fwd+bwd throughput (BASELINE.json metric) on B200.

Default workload = config 2 (BASELINE.json configs[1]): the CLIP ViT-Huge MLP block,
fc1 1280->5120 and fc2 5120->1280, 256 images x 257 tokens = 65792 tokens per GPU,
SwitchBack int8 (row-wise X/G, tensor-wise W) forward + input gradient on tcgen05
kind::i8, bf16 weight gradient on tcgen05 kind::f16. One step = forward + backward of
the two chained linears (the reference's switchback_fwd_bwd unit, bench.cpp:75-81, applied
to the MLP block of model.cpp:324-329 / 351-360 without its GELU): fc2 consumes fc1's
output, fc1's output gradient is fc2's input gradient; synthetic bf16 X and block-output
gradient G. N > 1: weak scaling, each rank owns 65792 tokens; dW all-reduce (NCCL) is the
only collective.

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
WORKLOAD = ("CLIP ViT-Huge MLP block 1280->5120->1280 (fc1 -> fc2 chained), 256 images x 257 tokens, "
            "int8 fwd/dX + bf16 dW")
# BASELINE.json configs as bench modes (--config); c2 is the headline line the driver runs.
CONFIGS = {
    "c2": (LAYERS, WORKLOAD, "switchback", "int8"),
    "c3": ([("qkv", 1280, 3840), ("out", 1280, 1280), ("fc1", 1280, 5120), ("fc2", 5120, 1280)],
           "All CLIP ViT-Huge linears of one block (qkv 1280->3840, out 1280->1280, fc1, fc2), 65792 tokens per GPU",
           "switchback", "int8"),
    "c4q": (LAYERS, "ViT-Huge MLP block, SwitchBackQ (row-wise W, row x row int8 dequant)", "switchback_q", "int8"),
    "c4fp8": (LAYERS, "ViT-Huge MLP block, SwitchBack fp8 (e4m3 fwd, e5m2 grad, kind::f8f6f4)", "switchback", "fp8"),
}
INT8_PEAK_TOPS = 4500.0  # B200 dense int8 datasheet; tools/mma_rate.cu measures 4.47 POPS 2-CTA MMA issue


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
        pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
print("ready", flush=True)
out = []
import select
while not select.select([sys.stdin], [], [], 0.002)[0]:
    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
    out.append("%d %s" % (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), "".join("1" if r & b else "0" for b in bits)))
print(mx)
print("\n".join(out), flush=True)
"""


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: a separate NVML process
    polling every 2 ms (no GIL contention with the launching thread); nvidia-smi every 200 ms
    in a thread when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, [hw, hw_thermal, sw_thermal, sw_power] bools)
        self.source = None
        self._proc = None
        self._stop = threading.Event()
        self._t = None

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        f = [x.strip() for x in out.strip().split(",")]
        if len(f) == 6:
            self.samples.append((float(f[0]), float(f[1]), [x.lower() == "active" for x in f[2:]]))

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                self._sample_smi()
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        try:
            self._proc = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.index)], stdin=subprocess.PIPE,
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            if self._proc.stdout.readline().strip() != "ready":
                raise RuntimeError("sampler")
            self.source = "nvml"
        except Exception:
            if self._proc:
                self._proc.kill()
            self._proc = None
            self.source = "nvidia-smi"
            self._t = threading.Thread(target=self._run_smi, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._proc:
            try:
                out, _ = self._proc.communicate("stop\n", timeout=10)
                lines = out.strip().splitlines()
                mx = float(lines[0])
                for ln in lines[1:]:
                    mhz, fl = ln.split()
                    self.samples.append((float(mhz), mx, [c == "1" for c in fl]))
            except Exception:
                self._proc.kill()
        else:
            self._stop.set()
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "source": self.source}
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({self.NAMES[i] for s in self.samples for i in range(4) if s[2][i]})
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": self.samples[0][1], "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


# ----------------------------------------------------------------- CPU side
REF_SAMPLE_TOKENS = 8192  # the ViT-H configs are timed at T = 8192 and scaled linearly in T


class RefStep:
    """One bounded step of the UNMODIFIED reference (oracle/_ref: lowprec::linear_forward +
    linear_backward, {kSwitchBack, kInt8}) over the chained C2 linears (fc1 -> fc2 forward,
    fc2 -> fc1 backward), token rows sharded over the host threads (rows are independent,
    SPEC.md:301-302; dW partials summed in a fixed order). The oracle port stands in only when
    oracle/_ref was not built."""

    def __init__(self, tokens: int, threads: int | None = None):
        import numpy as np

        import oracle as O

        self.O = O
        self.kind = "reference" if O.ref_available() else "port"
        self.threads = (threads or os.cpu_count() or 1) if self.kind == "reference" else 1
        self.tokens = tokens
        (_, n, hd), (_, _, m) = LAYERS
        rng = np.random.default_rng(10)  # X, G ~ N(0, 1), W ~ N(0, 1/fan_in) (model.cpp:199-202)
        self.dims = (n, hd, m)
        self.x = rng.standard_normal((tokens, n)).astype(np.float32)
        self.w1 = (rng.standard_normal((hd, n)) / np.sqrt(n)).astype(np.float32)
        self.w2 = (rng.standard_normal((m, hd)) / np.sqrt(hd)).astype(np.float32)
        self.g = rng.standard_normal((tokens, m)).astype(np.float32)

    def run(self) -> float:
        n, hd, m = self.dims
        t0 = time.perf_counter()
        if self.kind == "reference":
            rc = self.O.ref().ref_switchback_mlp_fwd_bwd_threaded(self.x, self.w1, self.w2, self.g, self.tokens, n, hd,
                                                                  m, self.threads, None, None, None, None)
            assert rc == 0
        else:
            h = self.O.switchback_forward(self.x, self.w1)
            self.O.switchback_forward(h, self.w2)
            dh, _ = self.O.switchback_backward(h, self.w2, self.g)
            self.O.switchback_backward(self.x, self.w1, dh)
        return time.perf_counter() - t0

    def sample(self) -> str:
        return (f"{self.tokens} tokens (BASELINE.md §3 sample) through fc1 -> fc2 chained (1280->5120->1280) "
                f"SwitchBack int8 fwd+bwd per step, token rows sharded over {self.threads} threads; per-step time extrapolated "
                f"linearly to {T_PER_GPU} tokens (the reference's cost is linear in T: linear.cpp:43-51, "
                f"matrix.cpp:58-66)")


def cpu_reference_rate(tokens: int = REF_SAMPLE_TOKENS):
    """cpu_baseline of our arm: one warm-up pass, then one timed T = 8192 step. (tokens/s, cores, sample, kind)"""
    warm = RefStep(512)
    warm.run()
    rs = RefStep(tokens)
    dt = rs.run()
    return tokens / dt, rs.threads, rs.sample(), rs.kind


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref) on all host
    threads, same metric / unit / config as our arm. Each of the W warm-up and K timed steps is
    one T = 8192 sample of the C2 step; the tokens/s rate is exact for the sample and the
    per-step time is extrapolated linearly to T = 65792 (marked). If the projected run would
    exceed ~4 minutes (a box with few cores), the sample shrinks and says so."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    tokens = args.ref_tokens
    probe = RefStep(1024)
    probe.run()
    dt = probe.run()
    per_token = dt / 1024
    budget = 240.0
    n_steps = max(1, args.steps) + args.warmup
    if per_token * tokens * n_steps > budget:
        tokens = max(256, int(budget / n_steps / per_token) // 256 * 256)
    rs = RefStep(tokens)
    for _ in range(args.warmup):
        rs.run()
    times = [rs.run() for _ in range(max(1, args.steps))]
    v = tokens * len(times) / sum(times)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T_PER_GPU / v * 1000.0, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8+f32 (reference CPU)", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD + f" (CPU reference, {tokens}-token sample per step)",
                       "tokens_per_gpu": T_PER_GPU, "sample_tokens_per_step": tokens,
                       "sample_ms_per_step": 1000.0 * sum(times) / len(times)},
            "extrapolated": True,
            "extrapolation": f"ms_per_step = {T_PER_GPU} tokens / measured rate: the reference cost is linear in T",
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": rs.threads, "kind": rs.kind,
                             "sample": rs.sample()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU side
def dw_traffic(m, n, T, fused=False):
    """ncu DRAM bytes (read + write) of one dW GEMM launch of this shape, from the committed
    --set full captures (profiles/dw_gemm_traffic.json, keyed "m x n x T", "+gq" for the launch
    that also quantizes G); None if unmeasured."""
    prof = os.path.join(ROOT, "profiles", "dw_gemm_traffic.json")
    if not os.path.exists(prof):
        return None
    with open(prof) as f:
        d = json.load(f)
    e = d.get("launches", {}).get(f"{m}x{n}x{T}" + ("+gq" if fused else ""))
    return e["dram_bytes"] if e else None


class Op:
    """One kernel (or layer call) of the step: what it is, what it does per launch, where it runs."""

    def __init__(self, label, fn, cls, work, stream="main", join=False, ar=None):
        self.label, self.fn, self.cls, self.work = label, fn, cls, work
        self.stream, self.join, self.ar = stream, join, ar


def run_ours(args):
    import torch

    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200 import dp
    from paper_2304_13013_b200 import lowprec as L

    layers_cfg, workload, variant, fmt = CONFIGS[args.config]
    rank, world, local = dp.init_from_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    T = args.tokens
    mode = L.LinearMode({"switchback": A.SB_SWITCHBACK, "switchback_q": A.SB_SWITCHBACK_Q}[variant],
                        A.SB_INT8 if fmt == "int8" else A.SB_FP8)
    cmode = mode.c()
    plain = variant == "switchback" and fmt == "int8"  # the kernel-by-kernel SwitchBack int8 step
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)

    def randn(*shape, scale=1.0):
        return (torch.randn(*shape, device=dev, generator=gen) * scale).to(torch.bfloat16)

    def empty(*shape, dtype=torch.bfloat16):
        return torch.empty(*shape, device=dev, dtype=dtype)

    layers = []
    for name, n, m in layers_cfg:
        lay = {"name": name, "n": n, "m": m, "x": randn(T, n), "w": randn(m, n, scale=n ** -0.5), "g": randn(T, m),
               "y": empty(T, m), "dx": empty(T, n), "dw": empty(m, n, dtype=torch.float32), "ctx": A.LinearCtx(),
               "xq": empty(T, n, dtype=torch.int8), "xs": empty(T, dtype=torch.float32),
               "wq": empty(m, n, dtype=torch.int8), "wqt": empty(n, m, dtype=torch.int8),
               "wst": empty(1, dtype=torch.float32),
               "gq": empty(T, m, dtype=torch.int8), "gs": empty(T, dtype=torch.float32)}
        lay["ws"] = L._workspace(mode, T, n, m, dev)
        layers.append(lay)
    # --dw-comm fused: dW lives in a symmetric (peer-mapped) buffer and the dW GEMM's epilogue
    # reduce-scatters into the owner ranks' copies (sb_dp_wgrad_allreduce_fused: zero, barrier,
    # GEMM + reduce-scatter, barrier, all-gather of owned rows); NCCL calls inside it, so eager
    fused_comm = args.dw_comm == "fused" and plain and not args.unfused_gq
    if fused_comm:
        if world > 1 and torch.distributed.get_backend() != "nccl":
            raise SystemExit("--dw-comm fused needs the NCCL backend (its barriers and all-gather are NCCL)")
        args.no_graph = True
        comm0 = dp.NcclComm(A.handle(local), rank, world) if world > 1 else None
        for lay in layers:
            lay["sym"] = dp.SymmetricBuffer(A.handle(local), 4 * lay["m"] * lay["n"], rank, world, comm=comm0)
            lay["dw"] = lay["sym"].view((lay["m"], lay["n"]))
    chained = layers_cfg is LAYERS  # the MLP block: fc2 reads fc1's Y, fc1's G is fc2's dX
    if chained:
        layers[1]["x"] = layers[0]["y"]
        layers[0]["g"] = layers[1]["dx"]
    h = A.handle(local)
    P = L._p

    # The step, kernel by kernel, through the public C-ABI: per linear, quantize_rowwise(X),
    # quantize_tensorwise(W) (both layouts from one read), the int8 forward GEMM; then, last
    # layer first, quantize_rowwise(G), the bf16 dW GEMM and the int8 dX GEMM. These are the
    # launches sb_linear_forward / sb_linear_backward issue (checked equal after the timed
    # region); splitting them lets every kernel be timed inside the step. With overlap the
    # quantize of G runs on a side stream next to the one-wave dW GEMM (which leaves SMs idle)
    # and is joined before the dX GEMM: both only read G (linear.cpp:232-245). The first
    # layer's dW runs before its dX so that, under DP, the last dW all-reduce overlaps that dX.
    def q_x(l):
        A.check(h.lib.sb_quantize_rowwise(h.h, P(l["x"]), A.SB_BF16, T, l["n"], l["n"], P(l["xq"]), l["n"], P(l["xs"])))

    def q_w(l):
        A.check(h.lib.sb_quantize_tensorwise(h.h, P(l["w"]), A.SB_BF16, l["m"], l["n"], l["n"], P(l["wq"]), l["n"],
                                             P(l["wqt"]), l["m"], P(l["wst"])))

    def gemm_fwd(l):
        A.check(h.lib.sb_gemm_i8(h.h, P(l["xq"]), P(l["xs"]), P(l["wq"]), P(l["wst"]), A.SB_SCALE_ROW_TENSOR, T, l["m"],
                                 l["n"], P(l["y"]), A.SB_BF16, 0))

    def q_g(l):
        A.check(h.lib.sb_quantize_rowwise(h.h, P(l["g"]), A.SB_BF16, T, l["m"], l["m"], P(l["gq"]), l["m"], P(l["gs"])))

    def gemm_dx(l):
        A.check(h.lib.sb_gemm_i8(h.h, P(l["gq"]), P(l["gs"]), P(l["wqt"]), P(l["wst"]), A.SB_SCALE_ROW_TENSOR, T,
                                 l["n"], l["m"], P(l["dx"]), A.SB_BF16, 0))

    def dw_gemm(l):
        A.check(h.lib.sb_wgrad(h.h, P(l["g"]), P(l["x"]), A.SB_BF16, T, l["m"], l["n"], P(l["dw"]), 0, 0))

    def dw_fused_comm(l):  # dW GEMM + reduce-scatter epilogue + all-gather (world 1: the GEMM alone)
        A.check(h.lib.sb_dp_wgrad_allreduce_fused(h.h, P(l["g"]), P(l["x"]), A.SB_BF16, T, l["m"], l["n"], P(l["dw"]),
                                                  P(l["gq"]), l["m"], P(l["gs"])))

    def dw_gemm_gq(l):  # dW GEMM with quantize_rowwise(G) in the same launch
        A.check(h.lib.sb_wgrad_quantize_rowwise(h.h, P(l["g"]), P(l["x"]), A.SB_BF16, T, l["m"], l["n"], P(l["dw"]),
                                                P(l["gq"]), l["m"], P(l["gs"])))

    def layer_fwd(l):
        A.check(h.lib.sb_linear_forward(h.h, C.byref(cmode), P(l["x"]), P(l["w"]), A.SB_BF16, T, l["n"], l["m"],
                                        P(l["y"]), C.byref(l["ctx"]), P(l["ws"]), l["ws"].numel()))

    def layer_bwd(l):
        A.check(h.lib.sb_linear_backward(h.h, C.byref(cmode), C.byref(l["ctx"]), P(l["g"]), P(l["dx"]), P(l["dw"]), 0))

    # G's row-wise quantize: inside the dW launch (default: the dW kernel's idle warps do it while
    # the tensor cores stream the GEMM), or as its own kernel on a side stream (--unfused-gq), or
    # serially (--unfused-gq --no-overlap)
    fused_gq = plain and not args.unfused_gq
    overlap = plain and not args.no_overlap and not fused_gq
    # W's tensor-wise quantizes depend on no activation: with overlap both run on the side stream
    # at the start of the step, under the first layer's X quantize, and the first GEMM joins them
    w_side = plain and not args.no_overlap
    ops = []
    if w_side:
        for l in layers:
            ops.append(Op(f"{l['name']} quantize_tensorwise W {l['m']}x{l['n']} (+transpose)", lambda l=l: q_w(l),
                          "quantize", l["m"] * l["n"] * 4 + 4, stream="side"))
    for i, l in enumerate(layers):
        nm, n, m = l["name"], l["n"], l["m"]
        if plain:
            ops.append(Op(f"{nm} quantize_rowwise X {T}x{n}", lambda l=l: q_x(l), "quantize", T * n * 3 + 4 * T))
            if not w_side:
                ops.append(Op(f"{nm} quantize_tensorwise W {m}x{n} (+transpose)", lambda l=l: q_w(l), "quantize",
                              m * n * 4 + 4))
            ops.append(Op(f"{nm} int8 fwd GEMM M={T} N={m} K={n}", lambda l=l: gemm_fwd(l), "int8_gemm", 2 * T * m * n,
                          join=w_side and i == 0))
        else:
            ops.append(Op(f"{nm} linear_forward", lambda l=l: layer_fwd(l), "layer", 2 * T * m * n))
    for l in reversed(layers):
        nm, n, m = l["name"], l["n"], l["m"]
        if fused_comm:
            ops.append(Op(f"{nm} bf16 dW GEMM m={m} n={n} K={T} + quantize_rowwise G + reduce-scatter",
                          lambda l=l: dw_fused_comm(l), "dw_gemm", 2 * T * m * n))
            ops.append(Op(f"{nm} int8 dX GEMM M={T} N={n} K={m}", lambda l=l: gemm_dx(l), "int8_gemm", 2 * T * m * n))
        elif fused_gq:
            ops.append(Op(f"{nm} bf16 dW GEMM m={m} n={n} K={T} + quantize_rowwise G {T}x{m}",
                          lambda l=l: dw_gemm_gq(l), "dw_gemm", 2 * T * m * n, ar=l["dw"]))
            ops.append(Op(f"{nm} int8 dX GEMM M={T} N={n} K={m}", lambda l=l: gemm_dx(l), "int8_gemm", 2 * T * m * n))
        elif plain:
            ops.append(Op(f"{nm} quantize_rowwise G {T}x{m}", lambda l=l: q_g(l), "quantize", T * m * 3 + 4 * T,
                          stream="side" if overlap else "main"))
            ops.append(Op(f"{nm} bf16 dW GEMM m={m} n={n} K={T}", lambda l=l: dw_gemm(l), "dw_gemm", 2 * T * m * n,
                          ar=l["dw"]))
            ops.append(Op(f"{nm} int8 dX GEMM M={T} N={n} K={m}", lambda l=l: gemm_dx(l), "int8_gemm", 2 * T * m * n,
                          join=overlap))
        else:
            ops.append(Op(f"{nm} linear_backward", lambda l=l: layer_bwd(l), "layer", 4 * T * m * n, ar=l["dw"]))
    # graph chunks end where a dW all-reduce is issued (world > 1): NCCL runs between replays
    chunks, cur = [], []
    for op in ops:
        cur.append(op)
        if op.ar is not None and world > 1:
            chunks.append(cur)
            cur = []
    if cur:
        chunks.append(cur)

    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    # the dW all-reduce: the library's own NCCL communicator (sb_dp_init, csrc/dp.cu) when the
    # ranks run NCCL; torch.distributed only for the gloo test hook
    comm = None
    if world > 1 and torch.distributed.get_backend() == "nccl" and not fused_comm:
        comm = dp.NcclComm(h, rank, world)
    ar = dp.GradAllReduce(comm=comm)

    def enqueue(chunk, evs):
        """Launch one chunk on the current stream, recording an event after every kernel (and
        around the side-stream ones). evs: list to append (op, start_event, end_event) to."""
        cur_s = torch.cuda.current_stream(dev)
        prev = torch.cuda.Event(enable_timing=True, external=True)
        prev.record(cur_s)
        for op in chunk:
            if op.stream == "side":
                side.wait_stream(cur_s)
                a = torch.cuda.Event(enable_timing=True, external=True)
                b = torch.cuda.Event(enable_timing=True, external=True)
                with torch.cuda.stream(side):
                    h.bind_stream(side.cuda_stream)
                    a.record(side)
                    op.fn()
                    b.record(side)
                h.bind_stream(cur_s.cuda_stream)
                evs.append((op, a, b))
                continue
            if op.join:
                cur_s.wait_stream(side)
            op.fn()
            e = torch.cuda.Event(enable_timing=True, external=True)
            e.record(cur_s)
            evs.append((op, prev, e))
            prev = e

    # warmup (eager), counting our launches of one step
    h.bind_stream(stream.cuda_stream)
    for i in range(max(1, args.warmup)):
        l0 = h.launches()
        for c in chunks:
            enqueue(c, [])
        launches_per_step = h.launches() - l0
    torch.cuda.synchronize()
    # one graph per (step, chunk), each with its own events: every kernel of every timed step
    # is timed on the device inside the timed region, with no gaps added between kernels
    replicas = []  # [(graphs or None, evs)]
    for r in range(args.steps):
        evs, graphs = [], []
        if not args.no_graph:
            for c in chunks:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    h.bind_stream(torch.cuda.current_stream(dev).cuda_stream)
                    enqueue(c, evs)
                graphs.append(g)
            h.bind_stream(stream.cuda_stream)
        replicas.append((graphs, evs))
    if not args.no_graph:
        for g in replicas[0][0]:
            g.replay()
        torch.cuda.synchronize()

    def step(r):
        graphs, evs = replicas[r]
        for j, c in enumerate(chunks):
            if graphs:
                graphs[j].replay()
            else:
                enqueue(c, evs)
            if world > 1 and c[-1].ar is not None:
                ar.launch(c[-1].ar)
        ar.wait()

    if world > 1:
        torch.distributed.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        start.record(stream)
        for r in range(args.steps):
            step(r)
        end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = start.elapsed_time(end) / args.steps
    ms = dp.max_over_ranks(ms, dev)
    value = T * world / (ms / 1000.0)
    launches = launches_per_step * args.steps

    # ---- per-kernel evidence from the in-step events (mean over the timed steps)
    pk = peaks()
    per = {}
    for _, evs in replicas:
        for op, a, b in evs:
            per.setdefault(op.label, [op, 0.0])[1] += a.elapsed_time(b)
    kernels = []
    for label, (op, tot) in per.items():
        us = tot / args.steps * 1000.0
        row = {"op": label, "class": op.cls, "us": us, "stream": op.stream}
        if op.cls == "int8_gemm":
            row.update(tops=op.work / us / 1e6, peak_tops=INT8_PEAK_TOPS, frac=op.work / us / 1e6 / INT8_PEAK_TOPS)
        elif op.cls == "dw_gemm":
            row.update(tflops=op.work / us / 1e6, peak_tflops=pk["bf16_tflops"],
                       frac=op.work / us / 1e6 / pk["bf16_tflops"])
        elif op.cls == "quantize":
            row.update(gbs=op.work / us / 1e3, peak_gbs=pk["hbm_gbs"], frac=op.work / us / 1e3 / pk["hbm_gbs"])
        kernels.append(row)
    step_us = ms * 1000.0
    cls_us = lambda c, main_only=False: sum(k["us"] for k in kernels  # noqa: E731
                                            if k["class"] == c and (not main_only or k["stream"] == "main"))
    int8_rows = [k for k in kernels if k["class"] == "int8_gemm"]
    summary = None
    if int8_rows:
        ops_tot = sum(per[k["op"]][0].work for k in int8_rows)
        t_tot = cls_us("int8_gemm")
        summary = {"int8_tops_in_step": ops_tot / t_tot / 1e6, "peak_tops": INT8_PEAK_TOPS,
                   "frac": ops_tot / t_tot / 1e6 / INT8_PEAK_TOPS,
                   "peak_source": "B200 dense int8 datasheet (4.5 POPS); MEASURED_PEAKS.json has no int8 entry",
                   # bench.cpp:83-89: (2 q_row + q_tensor + q_tt) / switchback_fwd_bwd
                   "quantize_fraction": cls_us("quantize") / step_us,
                   "quantize_fraction_critical_path": cls_us("quantize", True) / step_us,
                   "quantize_note": ("standalone quantize kernels only: G's row-wise quantize runs inside the dW "
                                     "GEMM launches (dw_gemm rows)") if fused_gq else "all quantize kernels",
                   "share_of_step": {c: cls_us(c) / step_us for c in ("int8_gemm", "dw_gemm", "quantize")},
                   "timing": "CUDA events recorded between kernels inside each step's graph, mean over the timed steps"}
    roof = None
    if plain:
        dw_rows = [k for k in kernels if k["class"] == "dw_gemm"]
        dw_us = sum(k["us"] for k in dw_rows)
        flops = sum(per[k["op"]][0].work for k in dw_rows)
        achieved = flops / dw_us / 1e6
        peak = pk["bf16_tflops"]
        trafs = [dw_traffic(l["m"], l["n"], T, fused_gq) for l in layers]
        roof = {"bound": "tensor",
                "kernel": "bf16 dW GEMM (tcgen05 kind::f16 cta_group::2, 256x384 one-wave tiles, MN-major operands)" +
                          (" with quantize_rowwise(G) in its idle warps (the launch's time includes it)"
                           if fused_gq else ""),
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": f"{pk['source']} bf16 burst (MEASURED_PEAKS.json bf16_tflops: the kernel is timed "
                               f"inside a {ms * args.steps:.0f} ms region); sustained figure "
                               f"{pk['bf16_tflops_sustained']}, datasheet dense 2250",
                "traffic": (sum(trafs) / len(trafs)) if all(t is not None for t in trafs) else None,
                "traffic_source": "profiles/dw_gemm_traffic.json (ncu --set full dram__bytes_read+write, per launch)",
                "algorithmic_bytes_per_launch": [2 * T * (l["m"] + l["n"]) + 4 * l["m"] * l["n"] +
                                                 ((T * l["m"] * 3 + 4 * T) if fused_gq else 0) for l in layers],
                "share_of_step": dw_us / step_us,
                "flops_per_launch": [2 * l["m"] * l["n"] * T for l in layers]}
    int8_ops_step = sum(4.0 * l["m"] * l["n"] * T for l in layers)

    # the decomposed step computes what the layer API computes (not timed)
    if plain:
        for l in layers[:1]:
            y0 = l["y"].clone()
            layer_fwd(l)
            torch.cuda.synchronize()
            assert torch.equal(y0, l["y"]), "kernel-by-kernel forward differs from sb_linear_forward"

    yard = cublas_yardstick(torch, layers, T, args) if rank == 0 else None
    e2e = None
    if not args.no_e2e and args.config == "c2":
        # every rank drives its own shard through the host entry (dW summed over ranks inside it
        # when the library communicator is up); whole-job rate = all tokens / slowest rank
        e2e = e2e_host(args, L, torch, world=world, dev=dev)
        if rank == 0 and world == 1:
            e2e["per_linear_entry"] = e2e_host_per_linear(args, L, torch)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "c2":
        r, cores, sample, kind = cpu_reference_rate()
        cpu = {"value": r, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None,
                "dtype": ("int8 (fwd, dX) + bf16 (dW), fp32 accumulate" if fmt == "int8" else
                          "fp8 e4m3/e5m2 (fwd, dX) + bf16 (dW), fp32 accumulate"),
                "data": "synthetic",
                "config": {"workload": workload, "config": args.config, "variant": variant, "format": fmt,
                           "tokens_per_gpu": T, "global_tokens": T * world,
                           "layers": [f"{n}->{m}" for _, n, m in layers_cfg], "parallelism": f"dp{world} (token shards)",
                           "l2": "inputs larger than L2 (X, G operands 168-673 MB each)",
                           "cuda_graphs": not args.no_graph,
                           "dw_comm": ("fused GEMM + peer reduce-scatter + all-gather" if fused_comm else
                                       "NCCL all-reduce on a comm stream") if world > 1 else None,
                           "g_quantize": ("fused into the dW GEMM launch (sb_wgrad_quantize_rowwise)" if fused_gq else
                                          "own kernel on a side stream next to the dW GEMM" if overlap else
                                          "own kernel, serial") if plain else "inside sb_linear_backward"},
                "gpu_launches": launches,
                "roofline": roof,
                "int8_tops_per_step": int8_ops_step / 1e12,
                "int8_summary": summary,
                "kernels": kernels,
                "clocks": clk.summary(),
                "e2e": e2e, "cpu_baseline": cpu, "yardstick_cublas_bf16": yard}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def adamw_traffic(n_params):
    """DRAM bytes of one optimizer step over n_params, scaled from the ncu measurement in
    profiles/adamw_traffic.json (None when absent)."""
    prof = os.path.join(ROOT, "profiles", "adamw_traffic.json")
    if not os.path.exists(prof):
        return None
    with open(prof) as f:
        d = json.load(f)
    return d["bytes_per_step"] / d["params"] * n_params


def run_c5(args):
    """BASELINE.json configs[4]: one StableAdamW step (optimizer.cpp:102-172, update_clip,
    beta1 0.9, beta2 0.99, eps 1e-6, weight decay 0.2) over the ~1.0e9 fp32 parameters of 51
    ViT-H blocks {3840x1280, 1280x1280, 5120x1280, 1280x5120}, whole
    tensors sharded over the ranks by size (dp.lpt_partition; strong scaling: total parameters
    fixed).
    HBM-bound: 28 B/param (read theta, g, v, u; write theta, v, u)."""
    import torch

    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200 import dp

    rank, world, local = dp.init_from_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shapes = [(3840, 1280), (1280, 1280), (5120, 1280), (1280, 5120)] * 51
    zero1 = args.zero1
    if zero1:
        # ZeRO-1: every tensor row-sharded by the fused reduce-scatter's ownership (dp.owned_rows),
        # one fp64 all-reduce of the 204 per-tensor RMS sums between the two phases
        rows = [dp.owned_rows(a, rank, world) for a, _ in shapes]
        mine = [(r1 - r0, b) for (r0, r1), (_, b) in zip(rows, shapes)]
    else:
        # whole tensors per rank, size-balanced (LPT: max / mean 1.0065 at 8 ranks; round-robin by
        # index was 1.36)
        mine = [shapes[i] for i in dp.lpt_partition([a * b for a, b in shapes], world)[rank]]
    total_params = sum(a * b for a, b in shapes)
    n_mine = sum(a * b for a, b in mine)
    # one flat allocation per state array, tensors are views (as a trainer's flat buffers)
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    flat = {k: torch.empty(n_mine, device=dev) for k in ("theta", "grad", "v", "u")}
    flat["theta"].normal_(generator=g).mul_(0.02)
    flat["grad"].normal_(generator=g).mul_(1e-3)
    flat["v"].zero_()
    flat["u"].zero_()
    arr = (A.AdamwTensor * len(mine))()
    off = 0
    for i, (a, b) in enumerate(mine):
        n = a * b
        arr[i] = A.AdamwTensor(*(flat[k].data_ptr() + 4 * off for k in ("theta", "grad", "v", "u")), n)
        off += n
    lib = A.load()
    nbytes = C.c_size_t()
    if zero1:
        A.check(lib.sb_stableadamw_sharded_workspace_size(arr, len(mine), C.byref(nbytes)))
        tot = (C.c_int64 * len(shapes))(*[a * b for a, b in shapes])
        comm = dp.NcclComm(A.handle(local), rank, world) if world > 1 and \
            torch.distributed.get_backend() == "nccl" else None
        if world > 1 and comm is None:
            raise SystemExit("--zero1 under N > 1 needs the NCCL backend (the library's fp64 all-reduce)")
    else:
        A.check(lib.sb_stableadamw_workspace_size(arr, len(mine), C.byref(nbytes)))
    ws = torch.empty(max(1, nbytes.value), dtype=torch.uint8, device=dev)
    out = torch.empty((2, len(mine)), dtype=torch.float64, device=dev)
    hp = A.AdamwHparams(1e-3, 0.9, 0.99, 0.0, 1e-6, 0.2, 1.0, A.SB_CLIP_UPDATE)
    h = A.handle(local)
    stream = torch.cuda.current_stream(dev)
    h.bind_stream(stream.cuda_stream)
    t = [0]

    def step():
        t[0] += 1
        if zero1:
            A.check(h.lib.sb_stableadamw_step_sharded(h.h, arr, tot, len(mine), C.byref(hp), t[0], None, None,
                                                      C.c_void_p(out[0].data_ptr()), C.c_void_p(out[1].data_ptr()),
                                                      C.c_void_p(ws.data_ptr()), ws.numel()))
            return
        A.check(h.lib.sb_stableadamw_step(h.h, arr, len(mine), C.byref(hp), t[0], C.c_void_p(out[0].data_ptr()),
                                          C.c_void_p(out[1].data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel()))

    for _ in range(max(3, args.warmup)):
        step()
    l0 = h.launches()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s_ev.record(stream)
        for _ in range(args.steps):
            step()
        e_ev.record(stream)
        torch.cuda.synchronize()
    launches = h.launches() - l0
    ms = dp.max_over_ranks(s_ev.elapsed_time(e_ev) / args.steps, dev)
    pk = peaks()
    achieved = 28.0 * n_mine / (ms / 1000.0) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_optimizer_rate()
    if rank == 0:
        line = {"metric": "StableAdamW step params/s over 1.0e9 ViT-H parameters (BASELINE.json configs[4])",
                "value": total_params / (ms / 1000.0), "unit": "params/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64 math / f32 storage", "data": "synthetic",
                "config": {"workload": "StableAdamW (update_clip) over 51 ViT-H blocks x 4 weight tensors",
                           "config": "c5", "params_total": total_params, "params_per_rank": n_mine,
                           "tensors_per_rank": len(mine),
                           "parallelism": (f"{world} ranks, ZeRO-1: every tensor row-sharded, phase 1 / fp64 "
                                           "all-reduce of the per-tensor RMS sums / phase 2") if zero1 else
                                          f"{world} ranks, whole tensors, size-balanced (LPT)",
                           "l2": "state (16 GB) far larger than L2"},
                "gpu_launches": launches,
                "roofline": {"bound": "hbm", "kernel": "StableAdamW phase 1 + 2 (csrc/optim.cu)", "achieved": achieved,
                             "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                             "traffic": None if zero1 else adamw_traffic(n_mine), "bytes_per_param": 28,
                             "note": ("ZeRO-1 splits the step at the RMS: phase 2 re-reads v, u from HBM (36 B/param "
                                      "moved, 28 counted)") if zero1 else None},
                "clocks": clk.summary(), "e2e": None, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_vit_block(args):
    """Model-level caller (model.cpp:287-408): one CLIP ViT-Huge
    transformer block (pre-LN; qkv 1280->3840, 16-head attention, out 1280->1280, fc1
    1280->5120, GELU, fc2 5120->1280; residuals), forward + backward at 256 x 257 tokens, with
    the four linears as paper_2304_13013_b200.nn.SwitchBackLinear (fp32 master weights, int8
    fwd/dX, bf16 dW) against the same block with torch bf16 linears under autocast (cuBLAS).
    LayerNorm, GELU and attention (SDPA) are PyTorch's in both arms. Each arm is captured in
    one CUDA graph; inputs and upstream gradients are synthetic and resident."""
    import torch
    import torch.nn.functional as F

    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200.nn import SwitchBackLinear, SwitchBackMLP

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B, S, D, H = 256, 257, 1280, 16
    fused = not args.no_overlap  # --no-overlap also turns the LayerNorm / GELU producer fusions off (A/B)
    # residual adds in the GEMM epilogues: SB_BLOCK_RESID=1 (measured slightly slower, 8.10-8.16 vs
    # 8.02-8.05 ms: the epilogue-heavy out-proj / fc2 GEMMs pay more for the extra reads)
    resid_fused = os.environ.get("SB_BLOCK_RESID", "0") == "1"
    T = B * S

    class SplitQKV(torch.autograd.Function):
        """q, k, v (B, H, S, Dh) views of the packed qkv output; the backward writes dq, dk, dv
        straight into one packed (B, S, 3, H, Dh) gradient (three strided copies) instead of
        autograd's stack + permute + contiguous (~1.9 ms of layout copies per step). Shared by
        both arms: it is block plumbing, not part of the measured linears."""

        @staticmethod
        def forward(ctx, qkv):
            t = qkv.view(B, S, 3, H, D // H)
            return tuple(t[:, :, i].transpose(1, 2) for i in range(3))

        @staticmethod
        def backward(ctx, dq, dk, dv):
            out = torch.empty(B, S, 3, H, D // H, dtype=dq.dtype, device=dq.device)
            for i, g in enumerate((dq, dk, dv)):
                out[:, :, i].copy_(g.transpose(1, 2))
            return out.view(B, S, 3 * D)

    class Block(torch.nn.Module):
        def __init__(self, sb):
            super().__init__()
            mk = (lambda i, o: SwitchBackLinear(i, o, device=dev)) if sb else \
                (lambda i, o: torch.nn.Linear(i, o, device=dev))
            self.ln1 = torch.nn.LayerNorm(D, device=dev)
            self.ln2 = torch.nn.LayerNorm(D, device=dev)
            self.fused = sb and fused
            self.out = mk(D, D)
            # q / k / v: three projections with their own tensor-wise scales as in the reference
            # block (model.cpp:303-305), run as one grouped GEMM; --qkv-packed quantizes the
            # packed [3D x D] weight with ONE scale instead (a numerics deviation, kept for A/B)
            groups = 1 if args.qkv_packed else 3
            if self.fused:
                # producer fusions: LayerNorm fused into the qkv / fc1 input quantization, GELU
                # into fc2's input quantization and fc1's gradient quantization
                self.qkv = SwitchBackLinear(D, 3 * D, device=dev, prenorm=True, groups=groups)
                self.mlp = SwitchBackMLP(D, 4 * D, device=dev, prenorm=True)
            elif sb:
                self.qkv = SwitchBackLinear(D, 3 * D, device=dev, groups=groups)
                fc1, fc2 = mk(D, 4 * D), mk(4 * D, D)
                self.mlp = torch.nn.Sequential(fc1, torch.nn.GELU(), fc2)
            else:
                self.qkv = mk(D, 3 * D)
                fc1, fc2 = mk(D, 4 * D), mk(4 * D, D)
                self.mlp = torch.nn.Sequential(fc1, torch.nn.GELU(), fc2)

        def forward(self, x):
            h = x if self.fused else self.ln1(x.float()).to(torch.bfloat16)
            if self.fused and not args.qkv_packed:
                # q / k / v handed to attention as head views; their gradients come back through
                # one pack + quantize kernel (SwitchBackLinear.qkv_heads)
                q, k, v = self.qkv.qkv_heads(h, H)
            else:
                q, k, v = SplitQKV.apply(self.qkv(h))
            a = F.scaled_dot_product_attention(q, k, v).transpose(1, 2).reshape(B, S, D)
            if self.fused and resid_fused:  # skip connections added in the out-proj / fc2 GEMM epilogues
                x = self.out(a, residual=x)
                return self.mlp(x, residual=x)
            x = x + self.out(a)
            h = x if self.fused else self.ln2(x.float()).to(torch.bfloat16)
            return x + self.mlp(h)

    gen = torch.Generator(device=dev).manual_seed(3)
    x0 = torch.randn(B, S, D, device=dev, generator=gen).to(torch.bfloat16)
    gy = torch.randn(B, S, D, device=dev, generator=gen).to(torch.bfloat16)
    res = {}
    launches = None
    for arm in ("switchback", "bf16"):
        blk = Block(arm == "switchback")
        x = x0.clone().requires_grad_(True)

        def step():
            for p in blk.parameters():
                p.grad = None
            x.grad = None
            with torch.autocast("cuda", dtype=torch.bfloat16, enabled=arm == "bf16"):
                y = blk(x)
            y.backward(gy)

        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
        torch.cuda.current_stream(dev).wait_stream(side)
        h = A.handle(0)
        l0 = h.launches()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        if arm == "switchback":
            launches = h.launches() - l0
        for _ in range(max(3, args.warmup)):
            g.replay()
        torch.cuda.synchronize()
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            s_ev.record()
            for _ in range(args.steps):
                g.replay()
            e_ev.record()
            torch.cuda.synchronize()
        ms = s_ev.elapsed_time(e_ev) / args.steps
        res[arm] = {"ms_per_step": ms, "value": T / (ms / 1000.0), "clocks": clk.summary()}
        if os.environ.get("SB_VIT_PROFILE"):  # kernel-time table of one replay on stderr (A/B aid, not the bench)
            from torch.profiler import ProfilerActivity, profile
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                g.replay()
                torch.cuda.synchronize()
            print(f"--- {arm} arm: one replay", file=sys.stderr)
            print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=90),
                  file=sys.stderr)
        del g, blk
        torch.cuda.empty_cache()
    sbv, bfv = res["switchback"], res["bf16"]
    line = {"metric": "ViT-H transformer block fwd+bwd tokens/s (model-level caller, SURVEY.md §8f row 2)",
            "value": sbv["value"], "unit": "tokens/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sbv["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int8 (linear fwd, dX) + bf16 (dW, attention, LN, GELU)", "data": "synthetic",
            "config": {"workload": "CLIP ViT-Huge block (pre-LN, 16-head SDPA, MLP 5120, GELU), 256 images x 257 tokens",
                       "config": "vit_block", "tokens": T, "cuda_graphs": True,
                       "l2": "activations far larger than L2"},
            "gpu_launches": launches * args.steps if launches is not None else None,
            "clocks": sbv["clocks"],
            "bf16_block": bfv, "speedup_vs_bf16_block": bfv["ms_per_step"] / sbv["ms_per_step"],
            "mlp_producer_fusion": fused,
            "qkv": "one packed weight, one tensor-wise scale (deviation)" if args.qkv_packed else
                   "three projections, three tensor-wise scales (model.cpp:303-305), one grouped GEMM",
            "e2e": None, "cpu_baseline": None, "roofline": None}
    print(json.dumps(line), flush=True)


def cpu_optimizer_rate(budget_s: float = 10.0):
    """The reference's optimizer_step (oracle/_ref, single-threaded as the reference) on a
    bounded sample of the C5 tensors; params/s."""
    import numpy as np

    import oracle as O

    if not O.ref_available():
        return None
    L = O.ref()
    shapes = [(1280, 1280), (3840, 1280)]
    rng = np.random.default_rng(0)
    arrs = [[(rng.standard_normal(a * b) * s).astype(np.float32) for s in (0.02, 1e-3, 0.0, 0.0)] for a, b in shapes]
    pp = C.POINTER(C.c_void_p)
    mk = lambda k: (C.c_void_p * len(arrs))(*[x[k].ctypes.data for x in arrs])  # noqa: E731
    numel = np.array([a * b for a, b in shapes], np.int64)
    rms, eta = np.zeros(len(shapes)), np.zeros(len(shapes))
    t0, n, t = time.perf_counter(), 0, 0
    while time.perf_counter() - t0 < budget_s:
        t += 1
        rc = L.ref_optimizer_step(len(shapes), C.cast(mk(0), pp), C.cast(mk(1), pp), C.cast(mk(2), pp),
                                  C.cast(mk(3), pp), numel, 1e-3, 0.9, 0.99, 0.0, 1e-6, 0.2, 1, 1.0, t, rms, eta)
        assert rc == 0
        n += int(numel.sum())
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "params/s", "cores": 1, "kind": "reference",
            "sample": f"{t} optimizer_step calls over 1280x1280 + 3840x1280 fp32 tensors (6.55 M params each), "
                      "lowprec::optimizer_step (single-threaded as the reference)"}


def e2e_host(args, L, torch, world=1, dev=None):
    """Same workload (the chained C2 MLP block) through the C-ABI host-buffer entry
    sb_switchback_mlp_fwd_bwd_host: pinned host X, W1, W2, G in; Y, dX, dW1, dW2 out, every
    step; the hidden activation and its gradient stay on the device (as in the device step).
    N > 1: every rank runs its shard concurrently (its own GPU and PCIe link), dW summed over the
    ranks inside the call; the time is the max over ranks."""
    from paper_2304_13013_b200 import _capi as A
    from paper_2304_13013_b200 import dp

    T = args.tokens
    (_, n, hd), (_, _, m) = LAYERS
    g = torch.Generator().manual_seed(7)
    x = torch.randn(T, n, generator=g).to(torch.bfloat16).pin_memory()
    w1 = (torch.randn(hd, n, generator=g) / n ** 0.5).to(torch.bfloat16).pin_memory()
    w2 = (torch.randn(m, hd, generator=g) / hd ** 0.5).to(torch.bfloat16).pin_memory()
    gg = torch.randn(T, m, generator=g).to(torch.bfloat16).pin_memory()
    h2d = (x.numel() + w1.numel() + w2.numel() + gg.numel()) * 2
    d2h = (T * m + T * n) * 2 + (w1.numel() + w2.numel()) * 4
    # >= 2 warm-up calls: the entry alternates two device pools, each allocated on first use
    for _ in range(max(3, args.warmup)):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, gg, A.SB_ACT_NONE)
    steps = max(10, args.steps)  # >= 10 calls: the PCIe rate of these hosts varies call to call
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, gg, A.SB_ACT_NONE)  # returns after Y, dX, dW1, dW2 are on the host
    torch.cuda.synchronize()
    dt = dp.max_over_ranks((time.perf_counter() - t0) / steps, dev)
    # informational: the async entry called back to back into two alternating preallocated output
    # sets (each call's uploads overlap the previous call's drain), one wait at the end
    outs = [tuple(torch.empty_like(t, pin_memory=True) for t in L.switchback_mlp_fwd_bwd_host(x, w1, w2, gg))
            for _ in range(2)]
    for i in range(2):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, gg, A.SB_ACT_NONE, wait=False, out=outs[i])
    L.host_pipeline_wait()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        L.switchback_mlp_fwd_bwd_host(x, w1, w2, gg, A.SB_ACT_NONE, wait=False, out=outs[i % 2])
    L.host_pipeline_wait()
    dt_async = dp.max_over_ranks((time.perf_counter() - t0) / steps, dev)
    return {"value": T * world / dt, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ranks": world,
            "pipelined_calls": {"value": T * world / dt_async, "unit": "tokens/s",
                                "note": "informational, not the headline: the async entry called back to back "
                                        "into two alternating output sets, each call's uploads overlapping the "
                                        "previous call's drain"},
            "path": "sb_switchback_mlp_fwd_bwd_host (C-ABI, pinned host buffers, 4096-token chunks: H2D / kernels / "
                    "D2H overlapped on three streams, hidden activation kept in HBM), one synchronous call per step",
            "pcie_note": "H2D and D2H share the link: 91-100 GB/s combined measured (tools/pcie_bw.py), so "
                         "the 752 MB of host traffic per step has a ~7.5-8.2 ms floor",
            "bytes_note": "h2d / d2h bytes are per rank and step", "steps": steps}


def e2e_host_per_linear(args, L, torch):
    """The per-linear host entry sb_switchback_fwd_bwd_host over both linears (X, W, G of each
    linear in; Y, dX, dW out): the hidden activation crosses PCIe four times. Secondary."""
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
    for _ in range(max(3, args.warmup)):  # both device pools allocated before the timed calls
        L.switchback_fwd_bwd_host_many(bufs)
    steps = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        L.switchback_fwd_bwd_host_many(bufs)  # both linears enqueued back to back, one wait
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return {"value": T / dt, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "path": "sb_switchback_fwd_bwd_host_async x 2 layers + sb_host_pipeline_wait (C-ABI, pinned host "
                    "buffers, chunked H2D/compute/D2H overlap, layer k+1 uploads overlap layer k's drain)",
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
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["c5", "vit_block"])
    ap.add_argument("--tokens", type=int, default=T_PER_GPU)
    ap.add_argument("--ref-tokens", type=int, default=REF_SAMPLE_TOKENS,
                    help="reference arm: token sample per step (BASELINE.md §3: 8192)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="one stream: W quantizes in line, G quantize after dW (with --unfused-gq)")
    ap.add_argument("--unfused-gq", action="store_true",
                    help="quantize G in its own kernel instead of inside the dW GEMM launch (A/B)")
    ap.add_argument("--qkv-packed", action="store_true", help="vit_block: one scale for the packed qkv weight")
    ap.add_argument("--zero1", action="store_true", help="c5: ZeRO-1 row-sharded optimizer (phase split + fp64 "
                    "all-reduce of the per-tensor RMS sums) instead of whole tensors per rank")
    ap.add_argument("--dw-comm", default="allreduce", choices=["allreduce", "fused"],
                    help="N > 1: NCCL all-reduce of dW after the GEMM on a comm stream (default), or the dW "
                         "GEMM's reduce-scatter epilogue over peer memory + all-gather (sb_dp_wgrad_allreduce_fused)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.config == "c5":
        run_c5(args)
    elif args.config == "vit_block":
        run_vit_block(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
