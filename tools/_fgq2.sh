timeout 300 python -m pytest tests/test_fused_wgrad_quant_gpu.py -x -q -k "matches_standalone" 2>&1 | grep -E "Error|error|assert|FAIL|passed|failed" | head -20
SB_DEBUG=1 timeout 120 python -c "
import torch
from paper_2304_13013_b200 import lowprec as L
g=torch.randn(65792,5120,device='cuda').bfloat16(); x=torch.randn(65792,1280,device='cuda').bfloat16()
try:
  L.wgrad_quantize_rowwise(g,x)
except Exception as e: print('ERR', e)
" 2>&1 | tail -5
