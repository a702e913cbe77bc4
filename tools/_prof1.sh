mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_dw_wide -s 4 -c 4 -o gpurun_out/prof_dwq -f python tools/prof_dwq.py > gpurun_out/prof_dwq.log 2>&1
tail -3 gpurun_out/prof_dwq.log
ls -la gpurun_out
