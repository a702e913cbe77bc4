timeout 600 python -m pytest tests/test_fused_wgrad_quant_gpu.py -q 2>&1 | tail -2
for w in 10 6; do
  SB_DWQ_WARPS=$w timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/fgq.json 2>gpurun_out/fgq.err
  python - "$w" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/fgq.json").read().strip().splitlines()[-1])
print("[w=%s]" % sys.argv[1], "ms/step %.3f" % d["ms_per_step"], "roof %.3f" % d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k in d["kernels"]:
    if "dW" in k["op"]: print("   %-70s %7.1f us" % (k["op"][:70], k["us"]))
PY
done
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_dw_wide -s 4 -c 4 -o gpurun_out/prof_dwq -f python tools/prof_dwq.py > gpurun_out/prof_dwq.log 2>&1
