#!/usr/bin/env bash
# A/B the int8 GEMM pipeline shapes inside the C2 step: in-step per-kernel times (bench.py
# --no-e2e --no-cpu) for each SB_GEMM_CFG value given on the command line.
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  SB_GEMM_CFG=$cfg python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_$cfg.json
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/ab_{sys.argv[1]}.json"))
print("cfg", sys.argv[1], "ms/step %.3f" % d["ms_per_step"], "int8 %.1f%%" % (100 * d["int8_summary"]["frac"]))
for k in d["kernels"]:
    if k["class"] in ("int8_gemm", "dw_gemm"):
        print("   %-45s %7.1f us  %.3f" % (k["op"], k["us"], k["frac"]))
PY
done
