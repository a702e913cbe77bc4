// tc_dw_wide.cuh — one-wave weight-gradient GEMM: dW = G^T X (linear.cpp:193-195) on
// cta_group::2 with 256 x 384 pair tiles, bf16 MN-major operands read in place (K = T tokens),
// fp32 raw accumulators stored once (no split-K, no memset, no reduce-add).
//
// Why: at the C2/C3 shapes the 256 x 256 tiling gives 100 tiles for 74 SM pairs, so the
// 2-CTA GEMM needs split-K = 2 (200 units, 2.7 waves, 90% wave efficiency, a 26 MB memset and
// fp32 reduce-adds). 256 x 384 tiles give 5 x 14 = 70 units: one wave, 95% of the pairs busy,
// every output element written once. For dW [5120 x 1280] the GEMM is run transposed
// (C = X^T G, M = n, N = m) and the epilogue writes C^T, so both MLP weight gradients map to
// 70 tiles.
//
// Per k-step of 16 tokens the leader issues two MMAs into one 384-column TMEM accumulator:
//   MMA a: N = 256 over B columns [0, 256)   (CTA r holds columns 128r .. 128r+127)
//   MMA b: N = 128 over B columns [256, 384) (CTA r holds columns 256+64r .. 256+64r+63)
// Stages hold 64 tokens: A 128 MN x 64 k (2 SW128 boxes), B 192 MN x 64 k (3 boxes) = 40 KB
// per CTA, 4 stages. Synchronisation as tc_gemm2.cuh (leader-only full barrier with both
// CTAs' bytes, multicast commits to both CTAs' empty barriers).
//
// Fused row-wise quantize of G (QV != 0). In SwitchBack's backward, G feeds both this GEMM (bf16)
// and the int8 dX GEMM (row-wise int8 G_q, linear.cpp:232-235). The dW kernel's epilogue warps
// sit idle through the whole main loop (one tile per pair, K = T tokens), and warps 2-3 always
// do; these 10 warps per CTA quantize G's rows (one warp per row, the standalone K1 row body,
// quant_core.cuh) while the producer / MMA threads stream the GEMM, so the quantize's HBM
// traffic overlaps tensor-core work inside one launch instead of competing for SMs from a
// second stream. QV = 16-byte vectors per lane in flight per step of the two-pass row quantizer
// (quant_core.cuh). The payload and states are those of sb_quantize_rowwise(G), bit for bit.
//
// Fused reduce-scatter (NM > 1, SURVEY.md §8e stage 2). Under token data parallelism dW is the
// sum over ranks of each rank's G_r^T X_r. With NM = 8 the kernel receives one D tensor map per
// rank, each over that rank's copy of a symmetric (CUDA-IPC peer-mapped) dW buffer, and every
// 32 x 32 output box leaves the epilogue as a TMA reduce-add (cp.reduce.async.bulk.tensor .add
// .f32) into the copy of the rank that owns its 32-row block of dW: the reduce-scatter's
// NVLink traffic streams out tile by tile while the tensor cores work, instead of a collective
// after the GEMM. Owned rows are then all-gathered (sb_dp_allgather_rows).
#pragma once
#include "quant_core.cuh"
#include "tc_gemm2.cuh"

namespace sbdw {

using namespace sbtc;
using sbtc2::cluster_sync;
using sbtc2::commit_mc;
using sbtc2::cta_rank;
using sbtc2::mbar_wait_cluster;
using sbtc2::tma_load_2sm;

constexpr int WN = 384;          // pair tile columns
constexpr int WM = 256;          // pair tile rows
constexpr int KROWS = 64;        // tokens per stage
constexpr int BOX = 8192;        // 64 MN x 64 k-rows bf16
constexpr int A_BYTES = 2 * BOX;
constexpr int B_BYTES = 3 * BOX;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NSTAGES = 4;
constexpr int SMEM_BYTES = NSTAGES * STAGE_BYTES + EPI_WARPS * EPI_BUF_BYTES + 1024 + 256;
static_assert(SMEM_BYTES <= MAX_DYN_SMEM, "shared memory budget");

struct WParams {
  int M, N, K;  // GEMM shape (TRANS: M = n, N = m)
  int tiles_m, tiles_n;
  // fused row-wise quantize of G [q_rows x 8 q_nvec] (QV != 0)
  const __nv_bfloat16* qg;
  int64_t q_rows, q_ld, q_ldq;  // rows, G row stride (elements), payload row stride (bytes)
  int q_nvec;                   // 16-byte vectors per row
  int8_t* q_out;
  float* q_state;
  uint32_t* q_err;
  int q_warps;  // quantizing warps per CTA: warps 2 .. 2 + q_warps - 1 (<= 2 + EPI_WARPS)
  int q_idle_kb;  // leading k-blocks of G quantized by the CTAs whose pair has no tile (unpaced)
  int q_lag;      // a working CTA quantizes k-block kb once its producer has issued kb + q_lag
};

// The quantize trails the GEMM through G: the GEMM streams G's rows (tokens) from HBM in
// k-blocks of 64 tokens, all pairs at about the same pace, and the quantize of a k-block's 64
// rows waits until this CTA's producer has issued the loads of k-block + kLag, so the rows are
// read from L2 (just brought in by the GEMM's TMA) instead of a second HBM stream racing the
// GEMM's own (measured: an unpaced quantize saturated HBM for its first ~150 us and stalled
// the GEMM). k-block kb belongs to working CTA kb mod (working CTAs); `prog` is the producer's
// progress (k-blocks issued), in shared memory. Lag sweep (C2 step, SB_DWQ_LAG): 48 / 24 / 12 /
// 6 / 2 / 0 k-blocks -> fc1 dW 717 / 702 / 694 / 691 / 689 / 685 us; -2 .. -16 (the quantize
// ahead of the producer) the same as 0 within noise; unpaced 847 us.
constexpr int kLag = 0;
constexpr int kQV = 8;  // vectors per lane in flight per step of the fused row quantizer
template <int QV>
__device__ __forceinline__ void quantize_g_rows(const WParams& p, int qwarp, int lane, const volatile int* prog,
                                                int k_blocks, int num_units) {
  if (qwarp >= p.q_warps) return;
  const int working = 2 * min(num_units, static_cast<int>(gridDim.x >> 1));  // CTAs whose pair has a tile
  const int c = static_cast<int>(blockIdx.x);
  const int qkb = static_cast<int>((p.q_rows + KROWS - 1) / KROWS);
  const bool idle = c >= working;
  // idle CTAs (no GEMM tile: every SM cycle is theirs) take the first q_idle_kb k-blocks at full
  // speed; the working CTAs take the rest, paced behind their own producer
  const int kb0 = idle ? c - working : p.q_idle_kb + c;
  const int kb_end = idle ? min(p.q_idle_kb, qkb) : qkb;
  const int kb_step = idle ? static_cast<int>(gridDim.x) - working : working;
  for (int kb = kb0; kb < kb_end; kb += kb_step) {
    const int need = min(kb + p.q_lag, k_blocks);
    while (!idle && *prog < need) __nanosleep(2000);
    const int64_t r1 = min(static_cast<int64_t>(kb + 1) * KROWS, p.q_rows);
#pragma unroll 1
    for (int64_t r = static_cast<int64_t>(kb) * KROWS + qwarp; r < r1; r += p.q_warps) {
      const uint4* xr = reinterpret_cast<const uint4*>(p.qg + r * p.q_ld);
      sbq::quantize_row_bf16_2pass<(QV > 0 ? QV : 1)>(xr, p.q_nvec, p.q_out + r * p.q_ldq, p.q_state + r, p.q_err, lane);
    }
  }
}

// The output tensor maps: NM = 1, the local dW (plain TMA store); NM = 8, one per rank's copy
// of the symmetric dW (TMA reduce-add into the owner of each 32-row block).
template <int NM>
struct DMaps {
  CUtensorMap m[NM];
  int world;    // ranks (<= NM)
  int nblocks;  // 32-row blocks of dW (ownership: block rb -> rank rb * world / nblocks)
};

__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(sbptx::smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void mma_f16_2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}

// TRANS: the accumulator row (GEMM row = n index) / column (m index) block of 32 x 32 is
// written to D[m][n] through a transposed staging tile: lane t (row t) stores its 32 values
// down column t of a [32 m][32 n] fp32 tile (SW128 layout of the D tensor map; for a fixed
// register index the 32 lanes fill one 128-byte row, so the stores are bank-conflict free).
template <bool TRANS, int QV, int NM = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_dw_wide(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ DMaps<NM> dm, const WParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + NSTAGES * A_BYTES;
  uint8_t* smem_epi = smem + NSTAGES * STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem_epi + EPI_WARPS * EPI_BUF_BYTES);
  uint64_t* empty_bar = full_bar + NSTAGES;
  uint64_t* tfull_bar = empty_bar + NSTAGES;
  uint64_t* tempty_bar = tfull_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 1);
  volatile int* prog = reinterpret_cast<volatile int*>(tmem_slot + 1);  // producer progress (k-blocks issued)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_units = p.tiles_m * p.tiles_n;
  const int k_blocks = (p.K + KROWS - 1) / KROWS;

  if (warp == 0 && lane == 0) {
    sbptx::tma_prefetch_desc(&tmA);
    sbptx::tma_prefetch_desc(&tmB);
    for (int r = 0; r < (NM > 1 ? dm.world : 1); ++r) sbptx::tma_prefetch_desc(&dm.m[r]);
    for (int s = 0; s < NSTAGES; ++s) {
      sbptx::mbar_init(&full_bar[s], 1);
      sbptx::mbar_init(&empty_bar[s], 1);
    }
    sbptx::mbar_init(tfull_bar, 1);
    sbptx::mbar_init(tempty_bar, 2 * EPI_WARPS);
    *prog = 0;
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
      const int m0 = (u % p.tiles_m) * WM, n0 = (u / p.tiles_m) * WN;
      const int am0 = m0 + static_cast<int>(rank) * BM;
      const int bn_a = n0 + static_cast<int>(rank) * 128;      // MMA a: 2 chunks of 64
      const int bn_b = n0 + 256 + static_cast<int>(rank) * 64;  // MMA b: 1 chunk
      for (int kb = 0; kb < k_blocks; ++kb) {
        sbptx::mbar_wait(&empty_bar[stage], phase ^ 1u);
        if (rank == 0) sbptx::mbar_arrive_expect_tx(&full_bar[stage], 2 * STAGE_BYTES);
        uint8_t* sa = smem_a + stage * A_BYTES;
        uint8_t* sb = smem_b + stage * B_BYTES;
        const int k0 = kb * KROWS;
        tma_load_2sm(&tmA, &full_bar[stage], sa, am0, k0);
        tma_load_2sm(&tmA, &full_bar[stage], sa + BOX, am0 + 64, k0);
        tma_load_2sm(&tmB, &full_bar[stage], sb, bn_a, k0);
        tma_load_2sm(&tmB, &full_bar[stage], sb + BOX, bn_a + 64, k0);
        tma_load_2sm(&tmB, &full_bar[stage], sb + 2 * BOX, bn_b, k0);
        if (QV != 0 && u == pair) *prog = kb + 1;  // first tile only: prog never goes back (no wait on a later tile)
        if (++stage == NSTAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // --------------------------------------------------------------- MMA issue (leader)
    if (rank == 0 && lane == 0) {
      // bf16 x bf16 -> f32, both operands MN-major, M = 256 (pair)
      const uint32_t id_a = sbptx::make_idesc(1, 1, 1, 1, 1, WM, 256);
      const uint32_t id_b = sbptx::make_idesc(1, 1, 1, 1, 1, WM, 128);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = pair; u < num_units; u += npairs, ++it) {
        mbar_wait_cluster(tempty_bar, (it & 1) ^ 1u);
        sbptx::tc_fence_after();
        for (int kb = 0; kb < k_blocks; ++kb) {
          sbptx::mbar_wait(&full_bar[stage], phase);
          sbptx::tc_fence_after();
          const uint32_t a_addr = sbptx::smem_u32(smem_a + stage * A_BYTES);
          const uint32_t b_addr = sbptx::smem_u32(smem_b + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < KROWS / 16; ++kk) {
            const uint64_t ad = sbptx::umma_desc_sw128(a_addr + kk * 2048, BOX, 1024);
            const uint32_t acc = (kb | kk) != 0;
            mma_f16_2(tmem_base, ad, sbptx::umma_desc_sw128(b_addr + kk * 2048, BOX, 1024), id_a, acc);
            mma_f16_2(tmem_base + 256, ad, sbptx::umma_desc_sw128(b_addr + 2 * BOX + kk * 2048, BOX, 1024), id_b,
                      acc);
          }
          commit_mc(&empty_bar[stage]);
          if (++stage == NSTAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        commit_mc(tfull_bar);
      }
    }
  } else if (warp == 2 || warp == 3) {
    if (QV != 0) quantize_g_rows<QV>(p, warp - 2, lane, prog, k_blocks, num_units);
  } else if (warp >= 4) {
    if (QV != 0) quantize_g_rows<QV>(p, warp - 2, lane, prog, k_blocks, num_units);
    // --------------------------------------------------------------- epilogue (both CTAs)
    const int ew = warp & 3;             // TMEM lane quarter
    const int half = (warp - 4) >> 2;    // column half: [192 half, 192 half + 192)
    uint8_t* buf = smem_epi + (warp - 4) * EPI_BUF_BYTES;
    int it = 0;
    for (int u = pair; u < num_units; u += npairs, ++it) {
      const int m0 = (u % p.tiles_m) * WM, n0 = (u / p.tiles_m) * WN;
      const int rm0 = m0 + static_cast<int>(rank) * BM + ew * 32;  // this warp's 32 GEMM rows
      sbptx::mbar_wait(tfull_bar, it & 1);
      sbptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + half * 192;
#pragma unroll 1
      for (int c = 0; c < 6; ++c) {  // 6 x 32 columns
        uint32_t r[32];
        sbptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
        sbptx::tmem_ld_wait();
        if (c == 5) {
          sbptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) sbtc::arrive_leader(tempty_bar);
        }
        const int col0 = n0 + half * 192 + c * 32;  // GEMM column of r[0]
        if (col0 >= p.N || rm0 >= p.M) continue;   // warp-uniform
        if (lane == 0) sbptx::tma_store_wait_read<0>();
        __syncwarp();
        if (TRANS) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int chunk = (lane >> 2) ^ (j & 7);
            *reinterpret_cast<uint32_t*>(buf + j * 128 + chunk * 16 + (lane & 3) * 4) = r[j];
          }
        } else {
          stage_row128(buf, lane, r);
        }
        sbptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          // D[m = col][n = row] (TRANS) or D[m = row][n = col]; c0 = n, c1 = m
          const int dn = TRANS ? rm0 : col0, dmr = TRANS ? col0 : rm0;
          if (NM > 1) {
            const int owner = static_cast<int>((static_cast<int64_t>(dmr >> 5) * dm.world) / dm.nblocks);
            tma_reduce_add_2d(&dm.m[owner], buf, dn, dmr);
          } else {
            sbptx::tma_store_2d(&dm.m[0], buf, dn, dmr);
          }
          sbptx::tma_store_commit();
        }
      }
    }
    if (lane == 0) {
      sbptx::tma_store_wait_all<0>();
      // the reduce-adds landed in peers' memory: make them visible system-wide before the
      // kernel (and the caller's barrier after it) completes
      if (NM > 1) __threadfence_system();
    }
  }
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    sbptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

}  // namespace sbdw
