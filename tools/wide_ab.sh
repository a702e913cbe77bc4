#!/usr/bin/env bash
# A/B the 256x384 int8 GEMM (SB_GEMM_WIDE=1) against the 256x256 one (0) inside the C2 step.
cd "$(dirname "$0")/.."
for w in "$@"; do
  SB_GEMM_WIDE=$w timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu ${BENCH_ARGS:-} > gpurun_out/wide_$w.json
  python - "$w" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/wide_{sys.argv[1]}.json"))
print("wide", sys.argv[1], "ms/step %.3f" % d["ms_per_step"], "int8 %.1f%%" % (100 * d["int8_summary"]["frac"]), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k in d["kernels"]:
    if k["class"] in ("int8_gemm", "dw_gemm"):
        print("   %-45s %7.1f us  %.3f" % (k["op"], k["us"], k["frac"]))
PY
done
