// feed_bench.cu — microbenchmark: how fast can TMA feed operand tiles L2 -> SMEM on all SMs?
// One producer lane per CTA streams K-major int8 tiles (box 128 B x ROWS) of a row-major
// [R x K] matrix into an S-stage ring; one consumer lane waits `full` and frees the slot.
// No MMA: this is the ceiling of the GEMM mainloop's operand feed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2304_13013_b200/csrc \
//   tools/feed_bench.cu paper_2304_13013_b200/csrc/gemm.cu -lcuda -o build/feed_bench
#include <cstdio>
#include <cstdlib>

#include "sb_internal.h"
#include "sb_ptx.cuh"

// wait variants: 0 try_wait (no hint), 1 try_wait + suspend-time hint, 2 test_wait spin
__device__ __forceinline__ void wait_v(uint64_t* bar, uint32_t parity, int v) {
  if (v == 0) {
    sbptx::mbar_wait(bar, parity);
  } else if (v == 1) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITH_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAITH_%=;\n\t}\n" ::"r"(sbptx::smem_u32(bar)), "r"(parity), "r"(0x989680)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAITT_%=;\n\t}\n" ::"r"(sbptx::smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__global__ void __launch_bounds__(64, 1) k_feed(const __grid_constant__ CUtensorMap tm, int rows_total, int kblocks,
                                                 int stages, int box_rows, int boxes, int iters, long long* out, const int8_t* src1d, int mode, int wv, long long* trace) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int stage_bytes = box_rows * 128 * boxes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      sbptx::mbar_init(&full[s], 1);
      sbptx::mbar_init(&empty[s], 1);
    }
    sbptx::fence_mbar_init();
  }
  __syncthreads();
  const int tiles_r = rows_total / (mode == 2 ? box_rows : box_rows * boxes);
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      const int tile = (blockIdx.x + i / kblocks * gridDim.x) % tiles_r;
      const int kb = i % kblocks;
      long long ta = clock64();
      wait_v(&empty[stage], ph ^ 1u, wv);
      long long tb = clock64();
      sbptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
      long long tc = clock64();
      if (mode == 0) {
        for (int b = 0; b < boxes; ++b)
          sbptx::tma_load_2d(&tm, &full[stage], smem + stage * stage_bytes + b * box_rows * 128, kb * 128,
                             (tile * boxes + b) * box_rows);
      } else if (mode == 2) {
        // one 3D box {128 B, box_rows, boxes K-atoms} per stage: dims (byte-in-atom, row, atom)
        const int atom0 = (kb * boxes) % (1280 / 128 - boxes + 1);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                sbptx::smem_u32(smem + stage * stage_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(tile * box_rows), "r"(atom0), "r"(sbptx::smem_u32(&full[stage]))
            : "memory");
      } else {
        for (int b = 0; b < boxes; ++b) {
          const int8_t* g = src1d + ((size_t)(tile * boxes + b) * box_rows * 1280 + (size_t)kb * box_rows * 128) % ((size_t)rows_total * 1280 - box_rows * 128);
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           sbptx::smem_u32(smem + stage * stage_bytes + b * box_rows * 128)),
                       "l"(g), "r"(box_rows * 128), "r"(sbptx::smem_u32(&full[stage]))
                       : "memory");
        }
      }
      if (blockIdx.x == 0 && i < 256) { long long td = clock64(); trace[2 * i] = td - t0; trace[600 + 3 * i] = tb - ta; trace[601 + 3 * i] = tc - tb; trace[602 + 3 * i] = td - tc; }
      if (++stage == stages) {
        stage = 0;
        ph ^= 1u;
      }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0;
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      wait_v(&full[stage], ph, wv);
      if (blockIdx.x == 0 && i < 256) { trace[2 * i + 1] = clock64() - t0; }
      sbptx::mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        ph ^= 1u;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 65536;  // rows of the source matrix
  const int K = 1280;
  int8_t* src;
  cudaMalloc(&src, (size_t)R * K);
  cudaMemset(src, 1, (size_t)R * K);
  long long* d;
  cudaMalloc(&d, 8 * 4096);
  long long* tr;
  cudaMalloc(&tr, 8 * 2048);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 2) sms = atoi(argv[2]);  // CTAs launched (one per SM): per-SM vs aggregate limit
  cudaFuncSetAttribute(k_feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  struct Cfg { int stages, box_rows, boxes, mode, per_sm, wv; };
  const Cfg cfgs[] = {{3, 128, 4, 0, 1, 0}, {3, 256, 2, 2, 1, 0}, {3, 128, 4, 2, 1, 0}, {6, 128, 2, 2, 1, 0}, {6, 128, 2, 0, 1, 0}};
  for (const Cfg& c : cfgs) {
    CUtensorMap tm;
    if (c.mode == 2) {
      // 3D view of the row-major [R x K] int8 matrix: (byte within a 128-B K atom, row, atom)
      const cuuint64_t dims[3] = {128, (cuuint64_t)R, (cuuint64_t)(K / 128)};
      const cuuint64_t strides[2] = {(cuuint64_t)K, 128};
      const cuuint32_t box[3] = {128, (cuuint32_t)c.box_rows, (cuuint32_t)c.boxes};
      const cuuint32_t estr[3] = {1, 1, 1};
      CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, src, dims, strides, box, estr,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("3D encode failed: %d\n", (int)r);
        continue;
      }
    } else if (!sb::encode_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, src, K, R, K, 128, c.box_rows,
                            CU_TENSOR_MAP_SWIZZLE_128B)) {
      printf("encode failed\n");
      return 1;
    }
    const int stage_bytes = c.box_rows * 128 * c.boxes;
    const int smem = c.stages * stage_bytes + 1024 + 512;
    if (smem * c.per_sm > 226 * 1024) continue;
    const int iters = 4000 * 49152 / stage_bytes;
    cudaEvent_t s, e;
    cudaEventCreate(&s);
    cudaEventCreate(&e);
    k_feed<<<sms * c.per_sm, 64, smem>>>(tm, R, K / 128, c.stages, c.box_rows, c.boxes, 100, d, src, c.mode, c.wv, tr);
    cudaEventRecord(s);
    k_feed<<<sms * c.per_sm, 64, smem>>>(tm, R, K / 128, c.stages, c.box_rows, c.boxes, iters, d, src, c.mode, c.wv, tr);
    cudaEventRecord(e);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, s, e);
    static long long h[4096];
    cudaMemcpy(h, d, 8 * sms * c.per_sm, cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < sms * c.per_sm; ++i) cyc += h[i];
    cyc /= sms * c.per_sm;
    const double bytes = (double)iters * stage_bytes * sms * c.per_sm;
    printf("wait=%d mode=%d ctas/SM=%d R=%d stages=%2d stage=%6d B (box %3d rows x %d)  err=%d  %.2f TB/s  %.1f B/clk/CTA  (%.0f MHz eff)\n", c.wv, c.mode, c.per_sm, R,
           c.stages, stage_bytes, c.box_rows, c.boxes, (int)err, bytes / (ms * 1e-3) / 1e12,
           (double)iters * stage_bytes / cyc, cyc / (ms * 1e-3) / 1e6);
    long long t[2048];
    cudaMemcpy(t, tr, 8 * 2048, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 64; ++i) printf("  i=%3d issue %7lld done %7lld  lat %6lld  wait %lld expect %lld tma %lld\n", i, t[2 * i], t[2 * i + 1], t[2 * i + 1] - t[2 * i], t[600 + 3 * i], t[601 + 3 * i], t[602 + 3 * i]);
  }
  return 0;
}
