mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -5
SB_GEMM_CFG=2 timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_fullsize_parity_gpu.py -x -q 2>&1 | tail -5
bash tools/gemm_ab.sh 0 2 2
