"""Step time with the step as 4 graph segments (bench.py) vs ONE graph, same kernels."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_13013_b200 import _capi as A, lowprec as L
T = 65792
dev = torch.device("cuda", 0)
mode = L.LinearMode(A.SB_SWITCHBACK, A.SB_INT8); cm = mode.c()
h = A.handle(0); P = L._p
lays = []
for n, m in [(1280, 5120), (5120, 1280)]:
    lay = dict(n=n, m=m, x=torch.randn(T, n, device=dev).bfloat16(), w=(torch.randn(m, n, device=dev) / n ** .5).bfloat16(),
               g=torch.randn(T, m, device=dev).bfloat16(), y=torch.empty(T, m, device=dev, dtype=torch.bfloat16),
               dx=torch.empty(T, n, device=dev, dtype=torch.bfloat16), dw=torch.empty(m, n, device=dev), ctx=A.LinearCtx())
    lay["ws"] = L._workspace(mode, T, n, m, dev)
    lays.append(lay)
def fwd(l):
    A.check(h.lib.sb_linear_forward(h.h, C.byref(cm), P(l["x"]), P(l["w"]), A.SB_BF16, T, l["n"], l["m"], P(l["y"]), C.byref(l["ctx"]), P(l["ws"]), l["ws"].numel()))
def bwd(l):
    A.check(h.lib.sb_linear_backward(h.h, C.byref(cm), C.byref(l["ctx"]), P(l["g"]), P(l["dx"]), P(l["dw"]), 0))
def step():
    fwd(lays[0]); fwd(lays[1]); bwd(lays[1]); bwd(lays[0])
segs = [lambda: (fwd(lays[0]), fwd(lays[1])), lambda: bwd(lays[1]), lambda: bwd(lays[0])]
for _ in range(3): step()
torch.cuda.synchronize()
g1 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g1):
    h.bind_stream(torch.cuda.current_stream().cuda_stream); step()
gs = []
for sgm in segs:
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.bind_stream(torch.cuda.current_stream().cuda_stream); sgm()
    gs.append(g)
def timeit(fn, k=20):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / k
for rep in range(2):
    print("one graph   %.3f ms" % timeit(g1.replay))
    print("3 segments  %.3f ms" % timeit(lambda: [g.replay() for g in gs]))
