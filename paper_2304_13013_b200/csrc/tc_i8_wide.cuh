// tc_i8_wide.cuh — the SwitchBack int8 GEMMs (forward Y = X_q W_q^T and input gradient
// dX = G_q (W_q^T)^T, linear.cpp:134 / :234-235) on cta_group::2 with 256 x 384 pair tiles,
// computed TRANSPOSED: C^T = W_q . X_q^T, so the 256-row side of a tile runs over weight rows
// (output columns: 1280 / 3840 / 5120 are multiples of 256) and the 384-wide side over tokens
// (T = 65792 = 171 x 384 + 128), and no shape of the ViT-H linears wastes MMA work on padding.
//
// Why 256 x 384: a 256 x 256 pair tile moves 64 KB per CTA per 256 bytes of K into shared memory
// (60.5 B/clk/SM at the dense int8 rate) and tops out at ~73% tensor-busy even with the output
// stores removed. 256 x 384 needs 17% fewer operand bytes per MMA op (49 B/clk/SM)
// and takes 40 KB stages of 128 bytes of K, 4 deep — the geometry of the one-wave bf16 dW kernel
// (tc_dw_wide.cuh), which runs 87-89% tensor-busy.
//
// Per k-step of 32 bytes the leader issues two MMAs (kind::i8 or kind::f8f6f4, M = 256):
//   MMA a: N = 256 over tokens [0, 256) of the tile   (CTA r holds tokens 128r .. 128r+127)
//   MMA b: N = 128 over tokens [256, 384)             (CTA r holds tokens 256+64r .. +63)
//
// TMEM (512 columns) cannot double-buffer a 384-column accumulator, so consecutive tiles
// alternate between two placements that overlap on 256 columns:
//   even tile: a -> [0, 256),   b -> [256, 384)
//   odd tile:  a -> [256, 512), b -> [0, 128)
// Tile t+1 reuses tile t's token columns [0, 128) and [256, 384) (the "early" set) plus the 128
// columns tile t did not use, which tile t-1 left behind in its columns [128, 256) (the "late"
// set). The epilogue drains each tile's early set first and signals `early`, then the late set
// (`late`); the MMA thread starts tile t+1 after early(t) and late(t-1). The next tile's MMAs
// therefore start as soon as two thirds of the accumulator are in registers, not after the
// whole epilogue.
//
// Epilogue (16 warps per CTA: TMEM lane quarter q = warp & 3 = 32 weight rows, token group g):
// group g drains its two early chunks of 32 tokens ({0,1}, {2,3}, {8,9}, {10,11}) with one pair
// of tcgen05.ld.32x32b.x32 (lane = weight row j, register k = token) and signals `early` at once,
// before converting anything; then its late chunk (4, 5, 6, 7) and `late`. The per-token scales
// are loaded before the accumulator is ready. (A first version with 8 epilogue warps, each
// converting and storing a pair of chunks before loading its second early pair, kept the MMA
// waiting on `early` 13-34% of the time: 300 / 421 us for the two C2 shapes.) The dequant y = f32(acc) * (s_token * 1/16129 * s_W) (+ bias_j) is
// the same fp32 arithmetic, in the same order, as the untransposed kernels (tc_gemm.cuh), so the
// outputs are bit-identical to them. bf16 outputs are transposed through one shuffle per two
// values into a [32 tokens][32 columns] staging block (conflict-free 4-byte stores) and written
// with a 2 KB TMA store; fp32 / int32 outputs store 128-byte rows directly.
#pragma once
#include "tc_gemm2.cuh"

namespace sbwide {

using namespace sbtc;
using sbtc2::cluster_sync;
using sbtc2::commit_mc;
using sbtc2::cta_rank;
using sbtc2::mbar_wait_cluster;
using sbtc2::tma_load_2sm;

constexpr int TW = 256;          // pair tile rows: weight rows (output columns)
constexpr int TT = 384;          // pair tile columns: tokens (output rows)
constexpr int KB = 128;          // bytes (= int8 / fp8 elements) of K per stage
constexpr int A_BYTES = 16384;   // 128 weight rows x 128 B
constexpr int B_BYTES = 24576;   // 128 + 64 token rows x 128 B
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NSTAGES = 4;
constexpr int EPI_BUF = 4096;    // per epilogue warp
constexpr int EPI_W = 16;        // epilogue warps: 4 TMEM lane quarters x 4 token groups
constexpr int THREADS = 128 + 32 * EPI_W;
constexpr int SMEM_BYTES = NSTAGES * STAGE_BYTES + EPI_W * EPI_BUF + 1024 + 256;
static_assert(SMEM_BYTES <= MAX_DYN_SMEM, "shared memory budget");

struct WideParams {
  int M;                 // tokens = output rows
  int N;                 // weight rows = output columns
  int K;
  const float* sa;       // per-token scale (X / G row states)
  const float* sb;       // per-weight-row (SB_COL) or tensor (one float) scale of W
  float post_scale;      // 1/16129 for int8, 1 for fp8
  const float* bias;     // optional, per output column (OUT_BF16 / OUT_F32)
  int tiles_w, tiles_t;  // weight tiles fast
};

template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == KIND_I8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}

// TMEM column of token chunk c (32 tokens) of tile iteration `it` (placement alternates).
__device__ __forceinline__ uint32_t chunk_col(int it, int c) {
  if ((it & 1) == 0) return static_cast<uint32_t>(32 * c);
  return c < 8 ? static_cast<uint32_t>(256 + 32 * c) : static_cast<uint32_t>(32 * (c - 8));
}

// One chunk: r[k] = accumulator of weight row j (this lane) and token i0 + k -> D[i0 + k][j];
// s = the scale of token i0 + lane.
template <int KIND, int OUT, bool SB_COL>
__device__ __forceinline__ void store_chunk(const WideParams& p, const CUtensorMap* tmD, uint32_t (&r)[32], int i0,
                                            int j0, int lane, uint8_t* buf, int& nst, float sbj, float bias_j,
                                            float sb_tensor, float s) {
  if (i0 >= p.M) return;  // warp-uniform: whole chunk past the last token
  if (OUT == OUT_BF16) {
    // the token factor exactly as tc_gemm.cuh forms it: (s * 1/16129) [* s_W tensor]
    const float fr = SB_COL ? s * p.post_scale : s * p.post_scale * sb_tensor;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const float fk = __shfl_sync(0xffffffffu, fr, k);
      float v = KIND == KIND_I8 ? i2f_exact(r[k]) : __uint_as_float(r[k]);
      v = SB_COL ? v * (fk * sbj) : v * fk;
      if (p.bias != nullptr) v = __fadd_rn(v, bias_j);
      r[k] = __float_as_uint(v);
    }
    uint8_t* b = buf + (nst & 1) * 2048;
    if (lane == 0) sbptx::tma_store_wait_read<1>();  // the store that last used this half is done reading
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const float lo = __uint_as_float(r[2 * m]), hi = __uint_as_float(r[2 * m + 1]);
      const float x = __shfl_xor_sync(0xffffffffu, (lane & 1) ? lo : hi, 1);
      const uint32_t w = (lane & 1) ? pack_bf16x2(x, hi) : pack_bf16x2(lo, x);
      // even lane: token 2m, columns (lane, lane + 1); odd lane: token 2m + 1, columns (lane - 1, lane)
      *reinterpret_cast<uint32_t*>(b + (2 * m + (lane & 1)) * 64 + (lane & ~1) * 2) = w;
    }
    sbptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      sbptx::tma_store_2d(tmD, b, j0, i0);
      sbptx::tma_store_commit();
    }
    ++nst;
  } else {
    const float fr = SB_COL ? s * p.post_scale : s * p.post_scale * sb_tensor;
    const float sw = SB_COL ? sbj : sb_tensor;
    if (lane == 0) sbptx::tma_store_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      uint32_t w;
      if (OUT == OUT_I32) {
        w = r[k];
      } else if (OUT == OUT_F32_EXACT) {  // float(double(acc) * sa_i * sb_j / 16129.0), linear.cpp:49
        const double sk = static_cast<double>(__shfl_sync(0xffffffffu, s, k));
        w = __float_as_uint(__double2float_rn(__ddiv_rn(
            __dmul_rn(__dmul_rn(static_cast<double>(static_cast<int32_t>(r[k])), sk), static_cast<double>(sw)),
            16129.0)));
      } else {
        const float fk = __shfl_sync(0xffffffffu, fr, k);
        const float v = KIND == KIND_I8 ? i2f_exact(r[k]) : __uint_as_float(r[k]);
        const float y = SB_COL ? __fmul_rn(v, fk * sbj) : __fmul_rn(v, fk);
        w = __float_as_uint(p.bias != nullptr ? __fadd_rn(y, bias_j) : y);
      }
      *reinterpret_cast<uint32_t*>(buf + k * 128 + lane * 4) = w;  // row = token k, column = j
    }
    sbptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      sbptx::tma_store_2d(tmD, buf, j0, i0);
      sbptx::tma_store_commit();
    }
  }
}

template <int KIND, int OUT, bool SB_COL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    k_gemm_wide(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmD, const WideParams p,
                uint32_t idesc_runtime) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + NSTAGES * A_BYTES;
  uint8_t* smem_epi = smem + NSTAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_epi + EPI_W * EPI_BUF);
  uint64_t* empty_bar = full_bar + NSTAGES;
  uint64_t* tfull_bar = empty_bar + NSTAGES;  // [2]
  uint64_t* early_bar = tfull_bar + 2;        // [2] leader only
  uint64_t* late_bar = early_bar + 2;         // [2] leader only
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(late_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_units = p.tiles_w * p.tiles_t;
  const int k_blocks = (p.K + KB - 1) / KB;

  if (warp == 0 && lane == 0) {
    sbptx::tma_prefetch_desc(&tmA);
    sbptx::tma_prefetch_desc(&tmB);
    sbptx::tma_prefetch_desc(&tmB2);
    sbptx::tma_prefetch_desc(&tmD);
    for (int s = 0; s < NSTAGES; ++s) {
      sbptx::mbar_init(&full_bar[s], 1);
      sbptx::mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sbptx::mbar_init(&tfull_bar[a], 1);
      sbptx::mbar_init(&early_bar[a], 2 * EPI_W);
      sbptx::mbar_init(&late_bar[a], 2 * EPI_W);
    }
    sbptx::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sbptx::smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  sbptx::tc_fence_before();
  __syncthreads();
  cluster_sync();
  sbptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  sbptx::pdl_trigger();
  sbptx::pdl_wait();

  if (warp == 0 && lane == 0) {
    // ---------------------------------------------------------------- producer (both CTAs)
    int stage = 0;
    uint32_t phase = 0;
    for (int u = pair; u < num_units; u += npairs) {
      const int w0 = (u % p.tiles_w) * TW + static_cast<int>(rank) * 128;
      const int t0 = (u / p.tiles_w) * TT;
      const int ta = t0 + static_cast<int>(rank) * 128, tb = t0 + 256 + static_cast<int>(rank) * 64;
      for (int kb = 0; kb < k_blocks; ++kb) {
        { SB_PROBE_T0(); sbptx::mbar_wait(&empty_bar[stage], phase ^ 1u); SB_PROBE_ADD(3); }
        if (rank == 0) sbptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
        uint8_t* sa = smem_a + stage * A_BYTES;
        uint8_t* sb = smem_b + stage * B_BYTES;
        tma_load_2sm(&tmA, &full_bar[stage], sa, kb * KB, w0);
        tma_load_2sm(&tmB, &full_bar[stage], sb, kb * KB, ta);
        tma_load_2sm(&tmB2, &full_bar[stage], sb + 16384, kb * KB, tb);
        if (++stage == NSTAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------------- MMA issue (leader)
    if (rank == 0 && lane == 0) {
      const uint32_t base = KIND == KIND_F8 ? idesc_runtime : sbptx::make_idesc(2, 1, 1, 0, 0, TW, 256);
      const uint32_t clr = ~((0x3Fu << 17) | (0x1Fu << 24));
      const uint32_t id_a = (base & clr) | ((256u >> 3) << 17) | ((static_cast<uint32_t>(TW) >> 4) << 24);
      const uint32_t id_b = (base & clr) | ((128u >> 3) << 17) | ((static_cast<uint32_t>(TW) >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
#ifdef SB_GEMM_PROBE
      const long long sb_loop0 = clock64(), sb_ns0 = gtime();
#endif
      for (int u = pair; u < num_units; u += npairs, ++it) {
        {
          SB_PROBE_T0();
          if (it >= 1) mbar_wait_cluster(&early_bar[(it - 1) & 1], ((it - 1) >> 1) & 1);
          if (it >= 2) mbar_wait_cluster(&late_bar[(it - 2) & 1], ((it - 2) >> 1) & 1);
          SB_PROBE_ADD(1);
        }
        sbptx::tc_fence_after();
        const uint32_t col_a = tmem_base + ((it & 1) ? 256u : 0u);
        const uint32_t col_b = tmem_base + ((it & 1) ? 0u : 256u);
        for (int kb = 0; kb < k_blocks; ++kb) {
          { SB_PROBE_T0(); sbptx::mbar_wait(&full_bar[stage], phase); SB_PROBE_ADD(0); }
          sbptx::tc_fence_after();
          const uint32_t a_addr = sbptx::smem_u32(smem_a + stage * A_BYTES);
          const uint32_t b_addr = sbptx::smem_u32(smem_b + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t ad = sbptx::umma_desc_sw128(a_addr + kk * 32, 16, 1024);
            const uint32_t acc = (kb | kk) != 0;
            mma<KIND>(col_a, ad, sbptx::umma_desc_sw128(b_addr + kk * 32, 16, 1024), id_a, acc);
            mma<KIND>(col_b, ad, sbptx::umma_desc_sw128(b_addr + 16384 + kk * 32, 16, 1024), id_b, acc);
          }
          commit_mc(&empty_bar[stage]);
          if (++stage == NSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        commit_mc(&tfull_bar[it & 1]);
      }
#ifdef SB_GEMM_PROBE
      atomicAdd(&g_probe[blockIdx.x * 6 + 2], (unsigned long long)(clock64() - sb_loop0));
      atomicAdd(&g_probe[blockIdx.x * 6 + 5], (unsigned long long)(gtime() - sb_ns0));  // loop ns (clock check)
#endif
    }
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue (both CTAs)
    const int q = warp & 3;
    const int g = (warp - 4) >> 2;
    uint8_t* buf = smem_epi + (warp - 4) * EPI_BUF;
    const float sb_tensor = SB_COL ? 1.0f : __ldg(p.sb);
    const int ce0 = g < 2 ? 2 * g : 4 + 2 * g;  // early pair {ce0, ce0 + 1}: {0,1} {2,3} {8,9} {10,11}
    const int cl = 4 + g;                        // late chunk
    int nst = 0;
    int it = 0;
    for (int u = pair; u < num_units; u += npairs, ++it) {
      const int j0 = (u % p.tiles_w) * TW + static_cast<int>(rank) * 128 + q * 32;  // weight row of lane 0
      const int t0 = (u / p.tiles_w) * TT;
      const int j = j0 + lane;
      // operand scales for this tile, fetched while the MMAs run
      const float sbj = (SB_COL && j < p.N) ? __ldg(p.sb + j) : 1.0f;
      const float bias_j = (p.bias != nullptr && j < p.N) ? __ldg(p.bias + j) : 0.0f;
      const int ia = t0 + 32 * ce0 + lane, ib = ia + 32, il = t0 + 32 * cl + lane;
      const float sa0 = ia < p.M ? __ldg(p.sa + ia) : 0.0f;
      const float sa1 = ib < p.M ? __ldg(p.sa + ib) : 0.0f;
      const float sal = il < p.M ? __ldg(p.sa + il) : 0.0f;
      { SB_PROBE_T0(); sbptx::mbar_wait(&tfull_bar[it & 1], (it >> 1) & 1); if (lane == 0 && warp == 4) SB_PROBE_ADD(4); }
      sbptx::tc_fence_after();
      const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      {
        uint32_t r0[32], r1[32];
        sbptx::tmem_ld_32x32b_x32(t_lane + chunk_col(it, ce0), r0);
        sbptx::tmem_ld_32x32b_x32(t_lane + chunk_col(it, ce0 + 1), r1);
        sbptx::tmem_ld_wait();
        sbptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&early_bar[it & 1]);
        if (j0 < p.N) {  // warp-uniform: rows past the last weight row store nothing
          store_chunk<KIND, OUT, SB_COL>(p, &tmD, r0, t0 + 32 * ce0, j0, lane, buf, nst, sbj, bias_j, sb_tensor, sa0);
          store_chunk<KIND, OUT, SB_COL>(p, &tmD, r1, t0 + 32 * ce0 + 32, j0, lane, buf, nst, sbj, bias_j, sb_tensor,
                                         sa1);
        }
      }
      {
        uint32_t r0[32];
        sbptx::tmem_ld_32x32b_x32(t_lane + chunk_col(it, cl), r0);
        sbptx::tmem_ld_wait();
        sbptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_leader(&late_bar[it & 1]);
        if (j0 < p.N)
          store_chunk<KIND, OUT, SB_COL>(p, &tmD, r0, t0 + 32 * cl, j0, lane, buf, nst, sbj, bias_j, sb_tensor, sal);
      }
    }
    if (lane == 0) sbptx::tma_store_wait_all<0>();
  }
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    sbptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

}  // namespace sbwide
