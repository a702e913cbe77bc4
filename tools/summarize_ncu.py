"""Summarize ncu captures (gpurun_out/*.ncu-rep, launches.csv) into profiles/ (committed).

    python tools/summarize_ncu.py r01
"""
import csv
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
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    r = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(r.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(hdr, units, vals):
        d[k] = (v, u)
    return d


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return x * scale


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    summary = {}
    for name in ("prof_dw", "prof_i8", "prof_q", "prof_k10", "prof_ln", "prof_lnb", "prof_adamw"):
        rep = os.path.join(OUT, name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        d = raw(rep)
        ent = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
        for k in KEYS:
            if k in d:
                ent[k] = {"value": d[k][0], "unit": d[k][1]}
        if "dram__bytes_read.sum" in d:
            ent["dram_bytes_total"] = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        summary[name] = ent
    if "prof_dw" in summary:
        with open(os.path.join(PROF, "dw_gemm_traffic.json"), "w") as f:
            json.dump({"kernel": summary["prof_dw"]["kernel"], "bytes_per_launch": summary["prof_dw"]["dram_bytes_total"],
                       "source": f"profiles/{tag}_ncu_summary.json (ncu --set full, one launch, fc2 dW)"}, f, indent=1)
    launches = []
    lp = os.path.join(OUT, "launches.csv")
    if os.path.exists(lp):
        rows = list(csv.reader(open(lp)))
        start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
        hdr = rows[start]
        idx = {k: i for i, k in enumerate(hdr)}
        for r in rows[start + 1:]:
            launches.append({"id": int(r[idx["ID"]]), "kernel": r[idx["Kernel Name"]][:90], "grid": r[idx["Grid Size"]],
                             "ns": float(r[idx["Metric Value"]].replace(",", ""))})
    with open(os.path.join(PROF, f"{tag}_ncu_summary.json"), "w") as f:
        json.dump({"captures": summary, "launches": launches}, f, indent=1)
    # human-readable launch list of one bench step (ours) next to the cuBLAS yardstick
    with open(os.path.join(PROF, f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list of `{os.environ.get('LAUNCH_CMD', 'python tools/prof_step.py')}`\n\n")
        f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` — cold-cache, serialised: compare shares.\n\n")
        f.write("| id | kernel | grid | us |\n|---|---|---|---|\n")
        for l in launches:
            f.write(f"| {l['id']} | `{l['kernel']}` | {l['grid']} | {l['ns'] / 1000:.1f} |\n")
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")
