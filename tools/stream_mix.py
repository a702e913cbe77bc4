"""HBM throughput vs the number of concurrent read / write streams (elementwise, float4,
grid-stride), to bound the StableAdamW kernel (3 read + 2 write streams in phase 1, 1-3 read +
1 write in phase 2). JIT-compiles one probe kernel (tool only, not part of the product).

    python tools/stream_mix.py
"""
import torch
from torch.utils.cpp_extension import load_inline

src = r"""
#include <torch/extension.h>
template <int R, int W>
__global__ void k(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                  float4* __restrict__ x, float4* __restrict__ y, float4* __restrict__ z, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    float4 s = __ldcs(a + i);
    if (R > 1) { float4 t = __ldcs(b + i); s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w; }
    if (R > 2) { float4 t = __ldcs(c + i); s.x += t.x; s.y += t.y; s.z += t.z; s.w += t.w; }
    __stcs(x + i, s);
    if (W > 1) __stcs(y + i, s);
    if (W > 2) __stcs(z + i, s);
  }
}
void run(int r, int w, torch::Tensor a, torch::Tensor b, torch::Tensor c, torch::Tensor x, torch::Tensor y,
         torch::Tensor z, int grid, int threads) {
  long n = a.numel() / 4;
  auto A = (const float4*)a.data_ptr<float>(); auto B = (const float4*)b.data_ptr<float>();
  auto C = (const float4*)c.data_ptr<float>(); auto X = (float4*)x.data_ptr<float>();
  auto Y = (float4*)y.data_ptr<float>(); auto Z = (float4*)z.data_ptr<float>();
#define L(RR, WW) if (r == RR && w == WW) k<RR, WW><<<grid, threads>>>(A, B, C, X, Y, Z, n);
  L(1,1) L(2,1) L(3,1) L(1,2) L(2,2) L(3,2) L(3,3) L(1,3)
}
"""
m = load_inline("stream_mix", cpp_sources="void run(int, int, torch::Tensor, torch::Tensor, torch::Tensor, torch::Tensor, torch::Tensor, torch::Tensor, int, int);",
                cuda_sources=src, functions=["run"], extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"],
                verbose=False)
n = 256 << 20
t = [torch.ones(n, device="cuda") for _ in range(6)]
sms = torch.cuda.get_device_properties(0).multi_processor_count
for r, w in [(1, 1), (2, 1), (3, 1), (1, 2), (2, 2), (3, 2), (1, 3), (3, 3)]:
    for occ in (4, 8, 16):
        grid = sms * occ
        for _ in range(2):
            m.run(r, w, *t, grid, 256)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            m.run(r, w, *t, grid, 256)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"R{r}W{w} blocks/SM {occ:2d}: {(r + w) * n * 4 / ms / 1e6:.0f} GB/s")
