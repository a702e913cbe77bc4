# Round-2 evidence under gpurun (PART=1|2|3 keeps each call's gpurun_out under the copy-back
# limit), then: python tools/summarize_r02.py
mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
F="--set full --clock-control none --import-source on"
case "${PART:-1}" in
1)
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
  tail -2 gpurun_out/pytest_gpu.txt
  timeout 400 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
  for c in c3 c4q c4fp8 c5 vit_block; do
    timeout 400 python bench.py --config $c --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  done
  timeout 400 python bench.py --config vit_block --no-overlap --no-cpu > gpurun_out/bench_vit_block_unfused.json 2>/dev/null
  timeout 400 python bench.py --unfused-gq --no-overlap --no-e2e --no-cpu > gpurun_out/bench_c2_unfused_gq.json 2>/dev/null
  timeout 400 python bench.py --dw-comm fused --no-e2e --no-cpu > gpurun_out/bench_c2_dw_comm_fused.json 2>/dev/null
  timeout 400 python bench.py --config c5 --zero1 --no-cpu > gpurun_out/bench_c5_zero1.json 2>/dev/null
  timeout 300 python tools/hbm_kernels.py > gpurun_out/hbm_kernels.txt 2>&1
  timeout 300 python tools/mlp_e2e_sweep.py 4096:0:2,4096:0:1,4096:0:0,8192:0:2,3072:0:2,6144:0:2 > gpurun_out/mlp_e2e_sweep.txt 2>&1
  timeout 300 python tools/e2e_timeline.py > gpurun_out/e2e_timeline.txt 2>&1
  timeout 300 python tools/pcie_bw.py > gpurun_out/pcie_bw.txt 2>&1
  timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
  timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_step.py > /dev/null 2>&1
  ;;
2)
  timeout 600 $N $F -k regex:k_dw_wide -s 4 -c 4 -o gpurun_out/prof_dwq -f python tools/prof_dwq.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:quantize_rowwise_reg -s 1 -c 1 -o gpurun_out/prof_q -f python tools/qprof.py > /dev/null 2>&1
  ;;
3)
  timeout 600 $N $F -k regex:k_tc_gemm2 -c 2 -o gpurun_out/prof_i8 -f python tools/gprof.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:tensorwise_coop -s 2 -c 1 -o gpurun_out/prof_tw -f python tools/twbench.py > /dev/null 2>&1
  ;;
4)
  timeout 600 $N $F -k regex:act_quantize_rows -s 2 -c 2 -o gpurun_out/prof_k10 -f python tools/prof_k10.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:k_ln_ -s 2 -c 2 -o gpurun_out/prof_ln -f python tools/prof_ln.py > /dev/null 2>&1
  NBLK=4 timeout 600 $N $F -k regex:adamw -s 2 -c 1 -o gpurun_out/prof_adamw -f python tools/oprof.py > /dev/null 2>&1
  timeout 600 $N $F -k regex:fp8_rows -s 1 -c 2 -o gpurun_out/prof_fp8 -f python tools/prof_fp8.py > /dev/null 2>&1
  ;;
esac
ls -la gpurun_out/
