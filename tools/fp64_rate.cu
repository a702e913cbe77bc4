// fp64_rate.cu — microbenchmark: DFMA / DDIV / DSQRT / F2F throughput per SM on this GPU
// (sizes the StableAdamW kernel's fp64 budget). nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
template <int OP>
__global__ void k(double* out, int iters, double a) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  float f[8];
  for (int j = 0; j < 8; ++j) f[j] = x[j];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) x[j] = __fma_rn(x[j], a, 1.0000001);
      if (OP == 1) x[j] = __ddiv_rn(a, x[j] + 1.0);
      if (OP == 2) x[j] = __dsqrt_rn(x[j] + 2.0);
      if (OP == 3) { f[j] = __double2float_rn(static_cast<double>(f[j]) * a); }
      if (OP == 4) x[j] = __dmul_rn(x[j], a);
    }
  }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j] + f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 148 * 8 * 1024 * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[] = {"DFMA", "DDIV", "DSQRT", "F2F f32->f64->f32 (+DMUL)", "DMUL"};
  for (int op = 0; op < 5; ++op) {
    int iters = op == 0 || op == 4 ? 4096 : 512;
    auto run = [&] {
      if (op == 0) k<0><<<sms * 8, 256>>>(d, iters, 0.9999999);
      if (op == 1) k<1><<<sms * 8, 256>>>(d, iters, 0.9999999);
      if (op == 2) k<2><<<sms * 8, 256>>>(d, iters, 0.9999999);
      if (op == 3) k<3><<<sms * 8, 256>>>(d, iters, 0.9999999);
      if (op == 4) k<4><<<sms * 8, 256>>>(d, iters, 0.9999999);
    };
    run();
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    cudaEventRecord(s);
    run();
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double ops = double(sms) * 8 * 256 * iters * 8;
    printf("%-28s %8.2f Gop/s  %6.2f op/clk/SM (at %d MHz nominal)\n", names[op], ops / (ms * 1e-3) / 1e9,
           ops / (ms * 1e-3) / (sms * clk * 1e3), clk / 1000);
  }
  return 0;
}
