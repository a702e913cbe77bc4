// gemm_probe.cu — run one tcgen05 GEMM shape with the SB_GEMM_PROBE pipeline counters and print
// where the MMA thread, the TMA producer and the epilogue spend their cycles.
// build: see tools/build_probe.sh
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../include/switchback_b200.h"
#include "../paper_2304_13013_b200/csrc/sb_internal.h"

extern "C" void sb_probe_read(unsigned long long* out, int n);

// pseudo-random operand bytes (realistic tensor-core power: constant data under-reports it)
__global__ void k_fill(uint8_t* p, size_t n, int bf16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ 0x9e3779b9u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    // bf16: keep exponents near 1.0 (0x3f00..0x3fff | sign) in the high byte of each element
    p[i] = bf16 ? ((i & 1) ? (uint8_t)(0x3f | (h & 0x80)) : (uint8_t)(h >> 8)) : (uint8_t)(h % 255 - 127 + 256);
  }
}
extern "C" void sb_probe_reset();
extern "C" void sb_probe_ns_read(unsigned long long* out, int n);
extern "C" void sb_trace_read(long long* out);

int main(int argc, char** argv) {
  const int64_t M = argc > 1 ? atoll(argv[1]) : 65792, N = argc > 2 ? atoll(argv[2]) : 5120,
                K = argc > 3 ? atoll(argv[3]) : 1280;
  const int kind = argc > 4 ? atoi(argv[4]) : 0;  // 0 int8 fwd, 1 bf16 dW (M=m, N=n, K=T)
  sb_handle h;
  if (sb_create(0, &h) != SB_OK) {
    printf("no device: %s\n", sb_last_error());
    return 1;
  }
  void *a, *b, *sa, *sbv, *out;
  const size_t esz = kind == 0 ? 1 : 2;
  cudaMalloc(&a, (kind == 0 ? M : K) * (kind == 0 ? K : M) * esz);
  cudaMalloc(&b, (kind == 0 ? N : K) * (kind == 0 ? K : N) * esz);
  cudaMalloc(&sa, M * 4);
  cudaMalloc(&sbv, 4);
  cudaMalloc(&out, M * N * 4);
  k_fill<<<1184, 256>>>((uint8_t*)a, (kind == 0 ? M * K : K * M) * esz, kind);
  k_fill<<<1184, 256>>>((uint8_t*)b, (kind == 0 ? N * K : K * N) * esz, kind);
  std::vector<float> ones(M, 1.0f);
  cudaMemcpy(sa, ones.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(sbv, ones.data(), 4, cudaMemcpyHostToDevice);
  auto run = [&] {
    if (kind == 0)
      return sb_gemm_i8(h, (int8_t*)a, (float*)sa, (int8_t*)b, (float*)sbv, SB_SCALE_ROW_TENSOR, M, N, K, out, SB_BF16, 0);
    return sb_wgrad(h, a, b, SB_BF16, K, M, N, (float*)out, 0, 0);
  };
  for (int i = 0; i < 3; ++i) run();
  cudaDeviceSynchronize();
  sb_probe_reset();
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  sb_status st = run();
  cudaEventRecord(e);
  cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  std::vector<unsigned long long> p(148 * 6);
  sb_probe_read(p.data(), 148 * 6);
  double sums[6] = {0};
  for (int c = 0; c < 148; ++c)
    for (int j = 0; j < 6; ++j) sums[j] += p[c * 6 + j];
  const double ops = 2.0 * M * N * K;
  printf("M=%lld N=%lld K=%lld kind=%d status=%d  %.1f us  %.0f T(FL)OPS\n", (long long)M, (long long)N, (long long)K, kind,
         st, ms * 1e3, ops / (ms * 1e-3) / 1e12);
  printf("per CTA avg (cycles): mma-loop %.0f | mma wait full %.0f | mma wait tempty %.0f | producer wait empty %.0f |"
         " epi(w4) wait tfull %.0f | k-blocks %.1f\n",
         sums[2] / 148, sums[0] / 148, sums[1] / 148, sums[3] / 148, sums[4] / 148, sums[5] / 148);
  if (getenv("TRACE")) {
    std::vector<long long> tr(4096);
    sb_trace_read(tr.data());
    const long long t0 = tr[1024];
    printf("stage: leader-issue peer-issue | mma-wait-begin mma-wait-end (ns from first wait)\n");
    for (int i = 0; i < 60; ++i)
      printf("%3d: %7lld %7lld | %7lld %7lld  wait %5lld\n", i, tr[i] - t0, tr[512 + i] - t0, tr[1024 + i] - t0,
             tr[1536 + i] - t0, tr[1536 + i] - tr[1024 + i]);
  }
  {
    std::vector<unsigned long long> ns(148);
    sb_probe_ns_read(ns.data(), 148);
    double cyc = 0, t = 0;
    for (int c = 0; c < 148; c += 2) t += ns[c];
    cyc = 2 * sums[2];
    if (t > 0) printf("256x256 kernel: MMA-loop %.0f cycles in %.0f ns per leader CTA -> %.0f MHz effective SM clock\n",
                      cyc / 74, t / 74, cyc / t * 1000.0);
  }
  if (getenv("SB_GEMM_WIDE") && atoi(getenv("SB_GEMM_WIDE")) == 1)
    printf("wide kernel: MMA-loop %.0f cycles in %.0f ns per leader CTA -> %.0f MHz effective SM clock\n",
           2 * sums[2] / 148, 2 * sums[5] / 148, sums[2] / sums[5] * 1000.0);
  printf("MMA busy fraction of loop ~ %.2f (ideal cycles = kblocks*4*128 = %.0f)\n",
         (sums[5] / 148 * 512) / (sums[2] / 148), sums[5] / 148 * 512);
  return 0;
}
