"""Quick read of one ncu report: time, DRAM bytes, pipe use, top stall reasons.

    python tools/ncu_quick.py gpurun_out/x.ncu-rep
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
r = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(r.splitlines()))
for row in rows[2:]:
    d = {k: (v, u) for k, u, v in zip(rows[0], rows[1], row)}
    print(d.get("Kernel Name", ("?",))[0][:90])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
              "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct"]:
        if k in d:
            print(f"  {k} {d[k][0]} {d[k][1]}")
    st = []
    for k, (v, u) in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print("  stalls:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:7]))
