// tc_gemm.cuh — persistent, warp-specialized tcgen05 GEMM for sm_100a.
//
//   D[M x N] = A . B^T, accumulated in TMEM, one 128 x 256 output tile per CTA at a time.
//
//   warp 0      TMA producer (one elected lane): A/B tiles -> 4-stage smem ring
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma, commits to mbarriers)
//   warps 4..7  epilogue: tcgen05.ld (32 lanes x 32 columns) -> scale/convert in registers ->
//               swizzled smem staging -> TMA store (or TMA reduce-add for accumulation)
//   Two TMEM accumulators (2 x 256 columns) let the epilogue of tile i overlap the MMAs of
//   tile i+1.
//
// Operand kinds:
//   KIND_I8   A, B int8 K-major (row-major [rows][K]); kind::i8, s32 accumulators.
//             SwitchBack forward Y = X_q . W_q^T and input gradient dX = G_q . (W_q^T)^T
//             (linear.cpp:134, :234-235).
//   KIND_F8   A, B e4m3/e5m2 K-major; kind::f8f6f4, f32 accumulators (linear.cpp:148-153).
//   KIND_BF16 bf16 operands, each either K-major or MN-major (A_MN / B_MN). The weight
//             gradient dW = G^T X (linear.cpp:193-195) reads G[T x m] and X[T x n] IN PLACE
//             as MN-major operands (K = T tokens) — no transposed copies. K-major/MN-major
//             mixes serve the Standard-mode linear (Y = X W^T, dX = G W).
#pragma once
#include <cuda_bf16.h>

#include "sb_ptx.cuh"

namespace sbtc {

enum Kind { KIND_I8 = 0, KIND_F8 = 1, KIND_BF16 = 2 };
enum Out {
  OUT_BF16 = 0,       // scaled, bf16
  OUT_F32 = 1,        // scaled, fp32 arithmetic
  OUT_F32_EXACT = 2,  // float(double(acc) * sa_i * sb_j / 16129.0)  (linear.cpp:49), int8 only
  OUT_I32 = 3,        // raw s32 accumulators
  OUT_F32_RAW = 4,    // raw f32 accumulators (dW), TMA store
  OUT_F32_RAW_ADD = 5 // raw f32 accumulators added into D (TMA reduce-add)
};

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = 16384;  // 128 rows x 128 B  (K-major)  |  64 k-rows x 128 elem x 2 B (MN)
constexpr int B_STAGE_BYTES = 32768;  // 256 rows x 128 B            |  64 k-rows x 256 elem x 2 B
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int EPI_BUF_BYTES = 4096;  // 32 rows x 128 B (f32/s32) or 32 rows x 64 B (bf16)
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 4 * 2 * EPI_BUF_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Params {
  int M, N, K;             // K in elements
  const float* sa;         // per-row (stride 1) or tensor (stride 0) state of A
  const float* sb;         // per-row-of-B (= per output column) or tensor state of B
  int sa_stride, sb_stride;
  float post_scale;        // 1/16129 for int8 dequant, 1 otherwise
  int tiles_m, tiles_n;
};

template <int KIND>
struct KindTraits;
template <>
struct KindTraits<KIND_I8> {
  static constexpr uint32_t IDESC = sbptx::make_idesc(2 /*s32*/, 1 /*s8*/, 1 /*s8*/, 0, 0, BM, BN);
  static constexpr int K_PER_STAGE = 128;  // elements (bytes)
};
template <>
struct KindTraits<KIND_F8> {
  // a/b formats patched at runtime (e4m3 = 0, e5m2 = 1)
  static constexpr uint32_t IDESC = sbptx::make_idesc(1 /*f32*/, 0, 0, 0, 0, BM, BN);
  static constexpr int K_PER_STAGE = 128;
};
template <>
struct KindTraits<KIND_BF16> {
  static constexpr uint32_t IDESC = sbptx::make_idesc(1 /*f32*/, 1 /*bf16*/, 1 /*bf16*/, 0, 0, BM, BN);
  static constexpr int K_PER_STAGE = 64;  // 64 bf16 = 128 B of K per stage
};

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Stage loader for one operand of `rows` (128 or 256) rows/cols.
//   K-major: one box {K_PER_STAGE elements (128 B), rows}      -> rows x 128 B, SW128
//   MN-major: rows/64 boxes {64 elements (128 B), 64 k-rows}   -> (rows/64) x 8 KB, SW128
template <bool MN, int KPS>
__device__ __forceinline__ void load_operand(const CUtensorMap* tm, uint64_t* bar, uint8_t* dst, int rows, int r0,
                                             int kb) {
  if (MN) {
    for (int j = 0; j < rows / 64; ++j) sbptx::tma_load_2d(tm, bar, dst + j * 8192, r0 + 64 * j, kb * 64);
  } else {
    sbptx::tma_load_2d(tm, bar, dst, kb * KPS, r0);
  }
}

// UMMA descriptor for MMA step k (of 4) within a stage.
//   K-major SW128: 128-byte rows, SBO = 8 rows (1 KB); one MMA consumes 32 bytes of K.
//   MN-major SW128: LBO = next 64-element MN chunk (8 KB), SBO = next 8 k-rows (1 KB);
//                   one MMA consumes 16 k-rows = 2 KB.
template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int k) {
  return MN ? sbptx::umma_desc_sw128(base + k * 2048, 8192, 1024) : sbptx::umma_desc_sw128(base + k * 32, 16, 1024);
}

template <int KIND, bool A_MN, bool B_MN, int OUT>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmD, const Params p, uint32_t idesc_runtime) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_STAGE_BYTES;
  uint8_t* smem_epi = smem + STAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_epi + 4 * 2 * EPI_BUF_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.tiles_m * p.tiles_n;
  const int k_blocks = (p.K + KindTraits<KIND>::K_PER_STAGE - 1) / KindTraits<KIND>::K_PER_STAGE;

  if (warp == 0 && lane == 0) {
    sbptx::tma_prefetch_desc(&tmA);
    sbptx::tma_prefetch_desc(&tmB);
    sbptx::tma_prefetch_desc(&tmD);
    for (int s = 0; s < STAGES; ++s) {
      sbptx::mbar_init(&full_bar[s], 1);
      sbptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sbptx::mbar_init(&tfull_bar[a], 1);
      sbptx::mbar_init(&tempty_bar[a], 4);
    }
    sbptx::fence_mbar_init();
  }
  if (warp == 1) sbptx::tmem_alloc(tmem_slot, TMEM_COLS);
  sbptx::tc_fence_before();
  __syncthreads();
  sbptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sbptx::mbar_wait(&empty_bar[stage], phase ^ 1u);
          sbptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE_BYTES);
          uint8_t* sa_ = smem_a + stage * A_STAGE_BYTES;
          uint8_t* sb_ = smem_b + stage * B_STAGE_BYTES;
          load_operand<A_MN, KindTraits<KIND>::K_PER_STAGE>(&tmA, &full_bar[stage], sa_, BM, m0, kb);
          load_operand<B_MN, KindTraits<KIND>::K_PER_STAGE>(&tmB, &full_bar[stage], sb_, BN, n0, kb);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issue
    if (lane == 0) {
      const uint32_t idesc = KIND == KIND_F8 ? idesc_runtime
                                             : (KindTraits<KIND>::IDESC | (A_MN ? (1u << 15) : 0u) | (B_MN ? (1u << 16) : 0u));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        sbptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
        sbptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sbptx::mbar_wait(&full_bar[stage], phase);
          sbptx::tc_fence_after();
          const uint32_t a_addr = sbptx::smem_u32(smem_a + stage * A_STAGE_BYTES);
          const uint32_t b_addr = sbptx::smem_u32(smem_b + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = operand_desc<A_MN>(a_addr, k);
            const uint64_t bd = operand_desc<B_MN>(b_addr, k);
            if (KIND == KIND_I8)
              sbptx::mma_i8(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else if (KIND == KIND_F8)
              sbptx::mma_f8(d_tmem, ad, bd, idesc, (kb | k) != 0);
            else
              sbptx::mma_f16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          sbptx::mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        sbptx::mma_commit(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    uint8_t* bufs = smem_epi + ew * 2 * EPI_BUF_BYTES;
    int bsel = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int m0 = (t / p.tiles_n) * BM, n0 = (t % p.tiles_n) * BN;
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      sbptx::mbar_wait(&tfull_bar[acc], acc_phase);
      sbptx::tc_fence_after();
      const int row = m0 + ew * 32 + lane;
      float row_scale = 1.0f;
      double row_scale_d = 1.0;
      if (OUT == OUT_BF16 || OUT == OUT_F32 || OUT == OUT_F32_EXACT) {
        const float s = row < p.M ? p.sa[p.sa_stride ? row : 0] : 0.0f;
        row_scale_d = static_cast<double>(s);
        row_scale = s * p.post_scale;
      }
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        sbptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        sbptx::tmem_ld_wait();
        if (c == BN / 32 - 1) {
          // accumulator fully drained into registers: hand TMEM back to the MMA warp
          sbptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) sbptx::mbar_arrive(&tempty_bar[acc]);
        }
        const int col0 = n0 + c * 32;
        if (col0 >= p.N) continue;  // whole chunk outside D (uniform across the warp)
        uint8_t* buf = bufs + bsel * EPI_BUF_BYTES;
        // make sure the TMA store that last used this buffer has finished reading it
        if (lane == 0) sbptx::tma_store_wait_read<1>();
        __syncwarp();
        if (OUT == OUT_BF16) {
          // 32 bf16 = 64 B per row; SWIZZLE_64B: 16-byte chunk j of row r lives at j ^ ((r >> 1) & 3)
          uint32_t w[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float v0, v1;
            const int ca = col0 + 2 * j, cb = ca + 1;
            float sb0 = 1.0f, sb1 = 1.0f;
            if (p.sb_stride) {
              sb0 = ca < p.N ? __ldg(p.sb + ca) : 0.0f;
              sb1 = cb < p.N ? __ldg(p.sb + cb) : 0.0f;
            } else {
              sb0 = sb1 = __ldg(p.sb);
            }
            if (KIND == KIND_I8) {
              v0 = static_cast<float>(static_cast<int32_t>(r[2 * j])) * row_scale * sb0;
              v1 = static_cast<float>(static_cast<int32_t>(r[2 * j + 1])) * row_scale * sb1;
            } else {
              v0 = __uint_as_float(r[2 * j]) * row_scale * sb0;
              v1 = __uint_as_float(r[2 * j + 1]) * row_scale * sb1;
            }
            w[j] = pack_bf16x2(v0, v1);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int pj = j ^ ((lane >> 1) & 3);
            *reinterpret_cast<uint4*>(buf + lane * 64 + pj * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
        } else {
          // 32 x 4-byte values = 128 B per row; SWIZZLE_128B: chunk j of row r at j ^ (r & 7)
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int cj = col0 + j;
            if (OUT == OUT_I32 || OUT == OUT_F32_RAW || OUT == OUT_F32_RAW_ADD) {
              w[j] = r[j];
            } else {
              const float sbj = p.sb_stride ? (cj < p.N ? __ldg(p.sb + cj) : 0.0f) : __ldg(p.sb);
              if (OUT == OUT_F32_EXACT) {
                const double d =
                    __ddiv_rn(__dmul_rn(__dmul_rn(static_cast<double>(static_cast<int32_t>(r[j])), row_scale_d),
                                        static_cast<double>(sbj)),
                              16129.0);
                w[j] = __float_as_uint(__double2float_rn(d));
              } else if (KIND == KIND_I8) {
                w[j] = __float_as_uint(static_cast<float>(static_cast<int32_t>(r[j])) * row_scale * sbj);
              } else {
                w[j] = __float_as_uint(__uint_as_float(r[j]) * row_scale * sbj);
              }
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int pj = j ^ (lane & 7);
            *reinterpret_cast<uint4*>(buf + lane * 128 + pj * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
          }
        }
        sbptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (OUT == OUT_F32_RAW_ADD) {
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmD)),
                "r"(sbptx::smem_u32(buf)), "r"(col0), "r"(m0 + ew * 32)
                : "memory");
          } else {
            sbptx::tma_store_2d(&tmD, buf, col0, m0 + ew * 32);
          }
          sbptx::tma_store_commit();
        }
        bsel ^= 1;
      }
    }
    if (lane == 0) sbptx::tma_store_wait_all<0>();
  }
  __syncthreads();
  if (warp == 1) {
    sbptx::tc_fence_after();
    sbptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

}  // namespace sbtc
