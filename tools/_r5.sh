timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_tc_gemm2 -c 2 -o gpurun_out/prof_i8 -f python tools/gprof.py > /dev/null 2>&1
ls -la gpurun_out/prof_i8.ncu-rep
