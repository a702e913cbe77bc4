timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_linear_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/b.json 2>gpurun_out/b.err; tail -3 gpurun_out/b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/b.json").read().strip().splitlines()[-1])
print("ms/step %.3f" % d["ms_per_step"], "roof %.3f" % d["roofline"]["frac"], "int8 %.3f" % d["int8_summary"]["frac"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for k in d["kernels"]: print("   %-70s %7.1f us" % (k["op"][:70], k["us"]))
PY
done
