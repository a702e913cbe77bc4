# ncu evidence for profiles/ (run under gpurun; PART=1 or PART=2 keeps each call's gpurun_out
# under the 64 MiB copy-back limit), then: python tools/summarize_ncu.py r01
mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
F="--set full --clock-control none --import-source on"
if [ "${PART:-1}" = "1" ]; then
  timeout 600 $N $F -k regex:k_tc_gemm2 -c 1 -o gpurun_out/prof_i8 -f python tools/gprof.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:k_dw_wide -c 1 -o gpurun_out/prof_dw -f python tools/gprof.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:quantize_rowwise_reg -s 1 -c 1 -o gpurun_out/prof_q -f python tools/qprof.py > /dev/null 2>&1
  timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
else
  timeout 600 $N $F -k regex:act_quantize_rows -s 2 -c 1 -o gpurun_out/prof_k10 -f python tools/prof_k10.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:k_ln_quantize -s 1 -c 1 -o gpurun_out/prof_ln -f python tools/prof_ln.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:k_ln_backward -s 1 -c 1 -o gpurun_out/prof_lnb -f python tools/prof_ln.py > /dev/null 2>&1
  NBLK=4 timeout 600 $N $F -k regex:adamw -s 2 -c 1 -o gpurun_out/prof_adamw -f python tools/oprof.py > /dev/null 2>&1
fi
ls -la gpurun_out/
