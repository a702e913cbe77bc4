"""Collect a round's GPU evidence from gpurun_out/ into profiles/ (committed).

    python tools/summarize_r02.py [tag]     (default r02)

* bench lines (gpurun_out/bench_*.json, last line)        -> profiles/<tag>_bench_<name>.json
* pytest -m gpu tail                                       -> profiles/<tag>_pytest_gpu_summary.txt
* ncu launch list (gpurun_out/launches.csv)                -> profiles/<tag>_launches.md
* ncu --set full reports (gpurun_out/prof_*.ncu-rep, every kernel in each report)
                                                           -> profiles/<tag>_ncu_summary.json
* dW DRAM bytes per launch, keyed m x n x T (+gq: with the fused G quantize)
                                                           -> profiles/dw_gemm_traffic.json (read by bench.py)
"""
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
NCU = "/usr/local/cuda/bin/ncu"
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def kernels_of(rep):
    r = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {k: (v, u) for k, u, v in zip(hdr, units, vals)}
        ent = {"kernel": d.get("Kernel Name", ("?", ""))[0][:120]}
        for k in KEYS:
            if k in d:
                ent[k] = {"value": d[k][0], "unit": d[k][1]}
        if "dram__bytes_read.sum" in d:
            ent["dram_bytes_total"] = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        stalls = []
        for k, (v, u) in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        ent["top_stalls_per_issue"] = {n: round(v, 2) for v, n in sorted(stalls, reverse=True)[:6]}
        out.append(ent)
    return out


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    for f in sorted(glob.glob(os.path.join(OUT, "bench_*.json"))):
        lines = [l for l in open(f).read().splitlines() if l.strip().startswith("{")]
        if lines:
            name = os.path.basename(f)[len("bench_"):-len(".json")]
            with open(os.path.join(PROF, f"{tag}_bench_{name}.json"), "w") as g:
                g.write(lines[-1] + "\n")
    pt = os.path.join(OUT, "pytest_gpu.txt")
    if os.path.exists(pt):
        tail = [l for l in open(pt).read().splitlines() if l.strip()][-3:]
        with open(os.path.join(PROF, f"{tag}_pytest_gpu_summary.txt"), "w") as g:
            g.write("python -m pytest tests -m gpu -q (one B200)\n" + "\n".join(tail) + "\n")
    summary = {}
    for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
        summary[os.path.basename(rep)[:-len(".ncu-rep")]] = kernels_of(rep)
    if summary:
        old = os.path.join(PROF, f"{tag}_ncu_summary.json")
        prev = json.load(open(old)) if os.path.exists(old) else {}
        prev.update(summary)
        with open(old, "w") as g:
            json.dump(prev, g, indent=1)
    if "prof_dwq" in summary and len(summary["prof_dwq"]) == 4:
        # tools/prof_dwq.py order: (m, n) = (5120, 1280), (1280, 5120); plain then fused each
        keys = ["5120x1280x65792", "5120x1280x65792+gq", "1280x5120x65792", "1280x5120x65792+gq"]
        tr = {"note": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per dW GEMM launch, keyed "
                      "m x n x T (+gq: the launch also quantizes G row-wise); read by bench.py dw_traffic",
              "launches": {k: {"dram_bytes": e["dram_bytes_total"], "kernel": e["kernel"][:40],
                               "source": f"profiles/{tag}_ncu_summary.json prof_dwq"}
                           for k, e in zip(keys, summary["prof_dwq"])}}
        with open(os.path.join(PROF, "dw_gemm_traffic.json"), "w") as g:
            json.dump(tr, g, indent=1)
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        rows = list(csv.reader(open(lp)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        idx = {k: i for i, k in enumerate(hdr)}
        launches = [{"id": int(r[idx["ID"]]), "kernel": r[idx["Kernel Name"]][:90], "grid": r[idx["Grid Size"]],
                     "ns": float(r[idx["Metric Value"]].replace(",", ""))} for r in rows[start + 1:] if len(r) > 5]
        with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as g:
            g.write(f"# {tag}: ncu launch list of `python tools/prof_step.py` (2 eager C2 bench steps, then the cuBLAS "
                    "yardstick)\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` — cold-cache, serialised: "
                    "compare shares, not absolute step times.\n\n| id | kernel | grid | us |\n|---|---|---|---|\n")
            for l in launches:
                g.write(f"| {l['id']} | `{l['kernel']}` | {l['grid']} | {l['ns'] / 1000:.1f} |\n")
    print("profiles updated:", sorted(os.listdir(PROF)))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
