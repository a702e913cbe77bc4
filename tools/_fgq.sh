mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_wgrad_quant_gpu.py tests/test_fullsize_parity_gpu.py tests/test_linear_gpu.py -x -q 2>&1 | tail -5
for a in "" "--unfused-gq" "--unfused-gq --no-overlap"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu $a > gpurun_out/fgq.json 2>gpurun_out/fgq.err
  python - "$a" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/fgq.json").read().strip().splitlines()[-1])
print("[%s]" % sys.argv[1], "ms/step %.3f" % d["ms_per_step"], "tok/s %.2fM" % (d["value"]/1e6), "roof %.3f" % d["roofline"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k in d["kernels"]:
    print("   %-70s %7.1f us  %s" % (k["op"][:70], k["us"], "%.3f" % k["frac"] if "frac" in k else ""))
PY
done
