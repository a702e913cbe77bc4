// tc_gemm2.cuh — the 2-CTA (cta_group::2) form of the persistent tcgen05 GEMM.
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile: CTA r loads its 128 rows of A
// and 128 of the 256 rows/cols of B; the leader (rank 0) issues tcgen05.mma.cta_group::2
// (M = 256), which reads A and B from both CTAs' shared memory and writes rows 0-127 of the
// accumulator to the leader's TMEM and rows 128-255 to the peer's. Per SM this halves the
// shared-memory operand bytes per MMA and the L2->SM operand traffic per flop relative to
// the 1-CTA 128 x 256 kernel (tc_gemm.cuh), and the 6-stage ring (32 KB / stage / CTA)
// doubles the K-depth in flight.
//
// Synchronisation (all mbarriers live at the same smem offsets in both CTAs):
//   full[s]   leader-only: 2 arrivals (leader arrive.expect_tx of both CTAs' bytes + the
//             peer's remote arrive); both CTAs' TMA loads complete_tx on the leader's copy.
//   empty[s]  per CTA: the leader's tcgen05.commit multicasts the arrival to both CTAs.
//   tfull[a]  per CTA: commit multicast when accumulator a is complete.
//   tempty[a] leader-only: 2 x 8 epilogue-warp arrivals (peer warps arrive remotely).
#pragma once
#include "tc_gemm.cuh"

namespace sbtc2 {

using namespace sbtc;

constexpr int STAGES2 = 6;
constexpr int A2_BYTES = 16384;  // per CTA: 128 rows x 128 B (K-major) | 64 k-rows x 128 elem x 2 B (MN)
constexpr int B2_BYTES = 16384;  // per CTA: half of B, same geometry
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr int BM2 = 256;         // tile rows per CTA pair
constexpr int SMEM2_BYTES = STAGES2 * STAGE2_BYTES + EPI_WARPS * EPI_BUF_BYTES + BN * 4 + 1024 + 512;
static_assert(SMEM2_BYTES <= MAX_DYN_SMEM, "shared memory budget");
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the CTA-rank bit of a shared::cluster address

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the leader CTA's copy of a barrier (works from either CTA)
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(sbptx::smem_u32(bar) & kPeerMask)
               : "memory");
}
__device__ __forceinline__ void tma_load_2sm(const CUtensorMap* m, uint64_t* bar, void* dst, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          sbptx::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(sbptx::smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void commit_mc(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          sbptx::smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// wait with cluster-scope acquire (the arrival comes from the peer CTA)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAITC_%=;\n\t}\n" ::"r"(sbptx::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
template <int KIND>
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == KIND_I8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  else if (KIND == KIND_F8)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}

// Work unit -> (m0 of the 256-row pair tile, n0, [kb0, kb1)).
__device__ __forceinline__ void unit2(const Params& p, int u, int k_blocks, int& m0, int& n0, int& kb0, int& kb1) {
  const int t = u / p.splits, s = u - t * p.splits;
  m0 = (p.m_fast ? t % p.tiles_m : t / p.tiles_n) * BM2;
  n0 = (p.m_fast ? t / p.tiles_m : t % p.tiles_n) * BN;
  kb0 = static_cast<int>((static_cast<int64_t>(k_blocks) * s) / p.splits);
  kb1 = static_cast<int>((static_cast<int64_t>(k_blocks) * (s + 1)) / p.splits);
}

template <int KIND, bool A_MN, bool B_MN, int OUT, bool SB_COL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_tc_gemm2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmD, const Params p, uint32_t idesc_runtime) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES2 * A2_BYTES;
  uint8_t* smem_epi = smem + STAGES2 * STAGE2_BYTES;
  float* col_scale = reinterpret_cast<float*>(smem_epi + EPI_WARPS * EPI_BUF_BYTES);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(col_scale + BN);
  uint64_t* empty_bar = full_bar + STAGES2;
  uint64_t* tfull_bar = empty_bar + STAGES2;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* pfull_bar = tempty_bar + 2;  // leader: "peer's stage landed" (relayed)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull_bar + STAGES2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_units = p.tiles_m * p.tiles_n * p.splits;
  constexpr int KPS = KindTraits<KIND>::K_PER_STAGE;
  const int k_blocks = (p.K + KPS - 1) / KPS;

  if (warp == 0 && lane == 0) {
    sbptx::tma_prefetch_desc(&tmA);
    sbptx::tma_prefetch_desc(&tmB);
    sbptx::tma_prefetch_desc(&tmD);
    for (int s = 0; s < STAGES2; ++s) {
      sbptx::mbar_init(&full_bar[s], 1);
      sbptx::mbar_init(&empty_bar[s], 1);
      sbptx::mbar_init(&pfull_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      sbptx::mbar_init(&tfull_bar[a], 1);
      sbptx::mbar_init(&tempty_bar[a], 2 * EPI_WARPS);
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
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / complete_tx
  sbptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < num_units; u += npairs) {
        int m0, n0, kb0, kb1;
        unit2(p, u, k_blocks, m0, n0, kb0, kb1);
        const int am0 = m0 + static_cast<int>(rank) * BM;         // this CTA's A rows
        const int bn0 = n0 + static_cast<int>(rank) * (BN / 2);   // this CTA's half of B
        for (int kb = kb0; kb < kb1; ++kb) {
          { SB_PROBE_T0(); sbptx::mbar_wait(&empty_bar[stage], phase ^ 1u); SB_PROBE_ADD(3); }
          // each CTA's loads complete on its OWN full barrier (plain 1-CTA TMA); the peer's
          // warp 1 relays completion to the leader (pfull) with one remote arrive
          sbptx::mbar_arrive_expect_tx(&full_bar[stage], STAGE2_BYTES);
          uint8_t* sa_ = smem_a + stage * A2_BYTES;
          uint8_t* sb_ = smem_b + stage * B2_BYTES;
          if (A_MN) {
            sbptx::tma_load_2d(&tmA, &full_bar[stage], sa_, am0, kb * 64);
            sbptx::tma_load_2d(&tmA, &full_bar[stage], sa_ + 8192, am0 + 64, kb * 64);
          } else {
            sbptx::tma_load_2d(&tmA, &full_bar[stage], sa_, kb * KPS, am0);
          }
          if (B_MN) {
            sbptx::tma_load_2d(&tmB, &full_bar[stage], sb_, bn0, kb * 64);
            sbptx::tma_load_2d(&tmB, &full_bar[stage], sb_ + 8192, bn0 + 64, kb * 64);
          } else {
            sbptx::tma_load_2d(&tmB, &full_bar[stage], sb_, kb * KPS, bn0);
          }
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issue (leader only)
    if (rank == 1 && lane == 0) {
      // relay: the peer's stage s landed -> arrive on the leader's pfull[s]
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < num_units; u += npairs) {
        int m0_, n0_, kb0, kb1;
        unit2(p, u, k_blocks, m0_, n0_, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          sbptx::mbar_wait(&full_bar[stage], phase);
          arrive_leader(&pfull_bar[stage]);
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
    if (rank == 0 && lane == 0) {
      const uint32_t base = KIND == KIND_F8 ? idesc_runtime : KindTraits<KIND>::IDESC;
      // M = 256 for the pair: m_dim field = 256 >> 4
      const uint32_t idesc = (base & ~(0x1Fu << 24)) | ((BM2 >> 4) << 24) | (A_MN ? (1u << 15) : 0u) |
                             (B_MN ? (1u << 16) : 0u);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = pair; u < num_units; u += npairs, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        { SB_PROBE_T0(); sbptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1u); SB_PROBE_ADD(1); }
        sbptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int m0_, n0_, kb0, kb1;
        unit2(p, u, k_blocks, m0_, n0_, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            SB_PROBE_T0();
            sbptx::mbar_wait(&full_bar[stage], phase);
            mbar_wait_cluster(&pfull_bar[stage], phase);
            SB_PROBE_ADD(0);
          }
#ifdef SB_GEMM_PROBE
          atomicAdd(&g_probe[blockIdx.x * 6 + 5], 1ull);
#endif
          sbptx::tc_fence_after();
          const uint32_t a_addr = sbptx::smem_u32(smem_a + stage * A2_BYTES);
          const uint32_t b_addr = sbptx::smem_u32(smem_b + stage * B2_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma2<KIND>(d_tmem, operand_desc<A_MN>(a_addr, k), operand_desc<B_MN>(b_addr, k), idesc, (kb != kb0) || k);
          commit_mc(&empty_bar[stage]);
          if (++stage == STAGES2) {
            stage = 0;
            phase ^= 1u;
          }
        }
        commit_mc(&tfull_bar[acc]);
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue (both CTAs)
    constexpr bool SCALED = OUT == OUT_BF16 || OUT == OUT_F32 || OUT == OUT_F32_EXACT;
    const int ew = warp & 3;
    const int half = (warp - 4) >> 2;
    const int ei = threadIdx.x - 128;
    uint8_t* buf = smem_epi + (warp - 4) * EPI_BUF_BYTES;
    const float sb_tensor = (SCALED && !SB_COL) ? __ldg(p.sb) : 1.0f;
    int it = 0;
    for (int u = pair; u < num_units; u += npairs, ++it) {
      int m0, n0, kb0_, kb1_;
      unit2(p, u, k_blocks, m0, n0, kb0_, kb1_);
      const int rm0 = m0 + static_cast<int>(rank) * BM;  // this CTA's 128 accumulator rows
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      float* cs = col_scale;
      if (SCALED && SB_COL) {
        epi_bar_sync();
        cs[ei] = (n0 + ei) < p.N ? __ldg(p.sb + n0 + ei) : 0.0f;
        epi_bar_sync();
      }
      const int row = rm0 + ew * 32 + lane;
      float fr = 1.0f;
      double sa_d = 1.0;
      if (SCALED) {
        const float s = row < p.M ? __ldg(p.sa + (p.sa_stride ? row : 0)) : 0.0f;
        sa_d = static_cast<double>(s);
        fr = SB_COL ? s * p.post_scale : s * p.post_scale * sb_tensor;
      }
      { SB_PROBE_T0(); sbptx::mbar_wait(&tfull_bar[acc], acc_phase); if (lane == 0 && warp == 4) SB_PROBE_ADD(4); }
      sbptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + half * 128;
#pragma unroll 1
      for (int pr = 0; pr < 2; ++pr) {
        uint32_t r0[32], r1[32];
        sbptx::tmem_ld_32x32b_x32(t_row + pr * 64, r0);
        sbptx::tmem_ld_32x32b_x32(t_row + pr * 64 + 32, r1);
        sbptx::tmem_ld_wait();
        if (pr == 1) {
          sbptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_leader(&tempty_bar[acc]);
        }
        const int cl = half * 128 + pr * 64;
        const int col0 = n0 + cl;
        if (col0 >= p.N || rm0 >= p.M) continue;
        if (OUT == OUT_BF16) {
          uint32_t w[32];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float a0, a1, b0, b1;
            if (KIND == KIND_I8) {
              a0 = static_cast<float>(static_cast<int32_t>(r0[2 * j]));
              a1 = static_cast<float>(static_cast<int32_t>(r0[2 * j + 1]));
              b0 = static_cast<float>(static_cast<int32_t>(r1[2 * j]));
              b1 = static_cast<float>(static_cast<int32_t>(r1[2 * j + 1]));
            } else {
              a0 = __uint_as_float(r0[2 * j]);
              a1 = __uint_as_float(r0[2 * j + 1]);
              b0 = __uint_as_float(r1[2 * j]);
              b1 = __uint_as_float(r1[2 * j + 1]);
            }
            if (SB_COL) {
              a0 *= fr * cs[cl + 2 * j];
              a1 *= fr * cs[cl + 2 * j + 1];
              b0 *= fr * cs[cl + 32 + 2 * j];
              b1 *= fr * cs[cl + 32 + 2 * j + 1];
            } else {
              a0 *= fr;
              a1 *= fr;
              b0 *= fr;
              b1 *= fr;
            }
            w[j] = pack_bf16x2(a0, a1);
            w[16 + j] = pack_bf16x2(b0, b1);
          }
          if (lane == 0) sbptx::tma_store_wait_read<0>();
          __syncwarp();
          stage_row128(buf, lane, w);
          sbptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sbptx::tma_store_2d(&tmD, buf, col0, rm0 + ew * 32);
            sbptx::tma_store_commit();
          }
        } else {
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            const uint32_t(&r)[32] = sub ? r1 : r0;
            const int cc = cl + sub * 32;
            if (n0 + cc >= p.N) break;
            uint32_t w[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (OUT == OUT_I32 || OUT == OUT_F32_RAW || OUT == OUT_F32_RAW_ADD) {
                w[j] = r[j];
              } else if (OUT == OUT_F32_EXACT) {
                const float sbj = SB_COL ? cs[cc + j] : sb_tensor;
                const double d = __ddiv_rn(
                    __dmul_rn(__dmul_rn(static_cast<double>(static_cast<int32_t>(r[j])), sa_d), static_cast<double>(sbj)),
                    16129.0);
                w[j] = __float_as_uint(__double2float_rn(d));
              } else {
                const float v = KIND == KIND_I8 ? static_cast<float>(static_cast<int32_t>(r[j])) : __uint_as_float(r[j]);
                w[j] = __float_as_uint(SB_COL ? v * (fr * cs[cc + j]) : v * fr);
              }
            }
            if (lane == 0) sbptx::tma_store_wait_read<0>();
            __syncwarp();
            stage_row128(buf, lane, w);
            sbptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if (OUT == OUT_F32_RAW_ADD) {
                asm volatile(
                    "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                        reinterpret_cast<uint64_t>(&tmD)),
                    "r"(sbptx::smem_u32(buf)), "r"(n0 + cc), "r"(rm0 + ew * 32)
                    : "memory");
              } else {
                sbptx::tma_store_2d(&tmD, buf, n0 + cc, rm0 + ew * 32);
              }
              sbptx::tma_store_commit();
            }
          }
        }
      }
    }
    if (lane == 0) sbptx::tma_store_wait_all<0>();
  }
  __syncthreads();
  cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    sbptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

}  // namespace sbtc2
