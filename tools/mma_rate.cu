// mma_rate.cu — microbenchmark: back-to-back tcgen05.mma issue rate (operands resident in
// smem, no TMA), 1-CTA M=128 vs 2-CTA M=256, kind::i8 and kind::f16, N=256 / 192 / 128.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o build/mma_rate
#include <cstdio>

#include "../paper_2304_13013_b200/csrc/tc_gemm2.cuh"

using namespace sbtc;

template <int KIND, bool TWO, int NN = 256>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, long long* out) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    sbptx::mbar_init(&bar, 1);
    sbptx::fence_mbar_init();
  }
  if (warp == 1) {
    if (TWO) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sbptx::smem_u32(&slot)), "r"(256));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      sbptx::tmem_alloc(&slot, 256);
    }
  }
  sbptx::fence_proxy_async_smem();
  sbptx::tc_fence_before();
  __syncthreads();
  if (TWO) sbtc2::cluster_sync();
  sbptx::tc_fence_after();
  const uint32_t tmem = slot;
  const bool leader = !TWO || sbtc2::cta_rank() == 0;
  if (warp == 1 && leader && (threadIdx.x & 31) == 0) {
    uint32_t idesc = KIND == KIND_I8 ? KindTraits<KIND_I8>::IDESC : KindTraits<KIND_BF16>::IDESC;
    if (TWO) idesc = (idesc & ~(0x1Fu << 24)) | (16u << 24);
    idesc = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(NN >> 3) << 17);
    const uint32_t a = sbptx::smem_u32(smem), b = sbptx::smem_u32(smem + 16384);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = operand_desc<false>(a, k), bd = operand_desc<false>(b, k);
        if (TWO)
          sbtc2::mma2<KIND>(tmem, ad, bd, idesc, 1);
        else if (KIND == KIND_I8)
          sbptx::mma_i8(tmem, ad, bd, idesc, 1);
        else
          sbptx::mma_f16(tmem, ad, bd, idesc, 1);
      }
    }
    if (TWO)
      sbtc2::commit_mc(&bar);
    else
      sbptx::mma_commit(&bar);
    sbptx::mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  } else if (TWO && warp == 1 && !leader && (threadIdx.x & 31) == 0) {
    sbptx::mbar_wait(&bar, 0);
  }
  __syncthreads();
  if (TWO) sbtc2::cluster_sync();
  if (warp == 1) {
    if (TWO)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    else
      sbptx::tmem_dealloc(tmem, 256);
  }
}

template <int KIND, bool TWO, int NN = 256>
void run(const char* name, int blocks) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 1024);
  cudaMemset(d, 0, sizeof(long long) * 1024);
  const int smem = 65536 + 2048;
  cudaFuncSetAttribute(k_rate<KIND, TWO, NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = TWO ? 2 : 1;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaLaunchKernelEx(&cfg, k_rate<KIND, TWO, NN>, iters, d);
  cudaEventRecord(s);
  cudaLaunchKernelEx(&cfg, k_rate<KIND, TWO, NN>, iters, d);
  cudaEventRecord(e);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, s, e);
  long long h[1024];
  cudaMemcpy(h, d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  const double mmas = 4.0 * iters;
  const double macs_per_mma = (TWO ? 256.0 : 128.0) * double(NN) * (KIND == KIND_I8 ? 32.0 : 16.0);
  const int issuers = TWO ? blocks / 2 : blocks;
  printf("%-22s blocks=%3d err=%d cyc/mma(leader0)=%.1f  chip=%.0f T%s/s\n", name, blocks, (int)err,
         double(h[0]) / mmas, issuers * mmas * macs_per_mma * 2.0 / (ms * 1e-3) / 1e12,
         KIND == KIND_I8 ? "OP" : "FLOP");
  cudaFree(d);
}

int main() {
  run<KIND_I8, false>("i8 1cta M128 N256", 1);
  run<KIND_I8, false>("i8 1cta M128 N256", 148);
  run<KIND_I8, true>("i8 2cta M256 N256", 2);
  run<KIND_I8, true>("i8 2cta M256 N256", 148);
  run<KIND_BF16, false>("bf16 1cta M128 N256", 148);
  run<KIND_BF16, true>("bf16 2cta M256 N256", 148);
  run<KIND_I8, true, 128>("i8 2cta M256 N128", 148);
  run<KIND_BF16, true, 128>("bf16 2cta M256 N128", 148);
  run<KIND_I8, true, 192>("i8 2cta M256 N192", 148);
  return 0;
}
