mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_quantize_gpu.py -q -x 2>&1 | tail -2
python tools/twbench.py
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_ln_quantize -s 1 -c 1 -o gpurun_out/prof_ln -f python tools/prof_ln.py > /dev/null 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:tensorwise_fused -s 2 -c 1 -o gpurun_out/prof_tw -f python tools/twbench.py > /dev/null 2>&1
ls gpurun_out
