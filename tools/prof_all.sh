set -x
mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
timeout 600 $N --set full --clock-control none --import-source on -k regex:k_tc_gemm2 -c 1 -o gpurun_out/prof_i8 -f python tools/gprof.py > /dev/null 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:k_dw_wide -c 1 -o gpurun_out/prof_dw -f python tools/gprof.py > /dev/null 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:quantize_rowwise_reg -s 1 -c 1 -o gpurun_out/prof_q -f python tools/qprof.py > /dev/null 2>&1
timeout 600 $N --set full --clock-control none --import-source on -k regex:act_quantize_rows -s 2 -c 1 -o gpurun_out/prof_k10 -f python tools/prof_k10.py > /dev/null 2>&1
NBLK=4 timeout 600 $N --set full --clock-control none --import-source on -k regex:adamw -s 2 -c 1 -o gpurun_out/prof_adamw -f python tools/oprof.py > /dev/null 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
ls -la gpurun_out/
