# quick GPU probe: each op once, small sizes, with hard sync after each
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
from paper_2304_13013_b200 import lowprec as L, _capi as A
def sync(name):
    torch.cuda.synchronize(); print("ok", name, flush=True)
x = torch.randn(256, 512, device='cuda')
q = L.quantize_rowwise(x); sync("rowwise")
qo, so = O.quantize(x.cpu().numpy(), O.ROW); print("rowwise exact", np.array_equal(q.payload.cpu().numpy(), qo))
w = torch.randn(384, 512, device='cuda')
qw, qwt = L.quantize_tensorwise(w, with_transpose=True); sync("tensorwise")
raw = L.int8_matmul_dequant(q, qw, out_dtype="raw"); sync("gemm raw")
want = q.payload.double().cpu() @ qw.payload.double().cpu().T
print("gemm raw exact", torch.equal(raw.double().cpu(), want), flush=True)
y = L.int8_matmul_dequant(q, qw, out_dtype=torch.bfloat16, exact=False); sync("gemm bf16")
g = torch.randn(1024, 256, device='cuda').bfloat16(); xx = torch.randn(1024, 512, device='cuda').bfloat16()
dw = L.wgrad(g, xx, exact=False); sync("wgrad")
ref = g.double().T @ xx.double()
print("wgrad rel", ((dw.double()-ref).norm()/ref.norm()).item(), flush=True)
