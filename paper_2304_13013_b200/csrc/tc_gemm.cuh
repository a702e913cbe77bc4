// tc_gemm.cuh — persistent, warp-specialized tcgen05 GEMM for sm_100a.
//
//   D[M x N] = A . B^T, accumulated in TMEM, one 128 x 256 output tile per CTA at a time.
//
//   warp 0       TMA producer (one lane): A/B tiles -> 4-stage smem ring (48 KB / stage)
//   warp 1       TMEM allocator + MMA issuer (one lane issues tcgen05.mma, commits to mbarriers)
//   warps 4..11  epilogue, 8 warps: warp w reads TMEM lane quarter (w & 3) and column half
//                ((w - 4) >> 2): tcgen05.ld 2 x (32 lanes x 32 columns) -> scale / convert in
//                registers -> 128B-swizzled smem staging -> TMA store (TMA reduce-add for
//                accumulation). Scales are hoisted: one per-row factor per tile, per-column
//                factors staged once per tile in smem.
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
  OUT_F32_RAW_ADD = 5, // raw f32 accumulators added into D (TMA reduce-add)
  OUT_BF16_RESID = 6   // scaled, + bias, + a bf16 residual tile (p.resid), rounded once to bf16
};

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int STAGES = 4;
constexpr int A_STAGE_BYTES = 16384;  // 128 rows x 128 B  (K-major)  |  64 k-rows x 128 elem x 2 B (MN)
constexpr int B_STAGE_BYTES = 32768;  // 256 rows x 128 B            |  64 k-rows x 256 elem x 2 B
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int EPI_WARPS = 8;
constexpr int EPI_BUF_BYTES = 4096;  // per epilogue warp: 32 rows x 128 B
constexpr int NUM_THREADS = 128 + 32 * EPI_WARPS;
constexpr int TMEM_COLS = 512;
constexpr int MAX_DYN_SMEM = 232448;  // 227 KB opt-in limit per CTA on sm_100
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_WARPS * EPI_BUF_BYTES + BN * 4 /*col scales*/ +
                           1024 /*align*/ + 256 /*barriers*/;
static_assert(SMEM_BYTES <= MAX_DYN_SMEM, "shared memory budget");

struct Params {
  int M, N, K;             // K in elements
  const float* sa;         // per-row (stride 1) or tensor (stride 0) state of A
  const float* sb;         // per-row-of-B (= per output column) or tensor state of B
  int sa_stride, sb_stride;
  float post_scale;        // 1/16129 for int8 dequant, 1 otherwise
  int tiles_m, tiles_n;
  int splits;              // split-K factor: work unit u = (tile u / splits, k-slice u % splits)
  int m_fast;              // raster: 1 = consecutive tiles walk M (B tile reused), 0 = walk N (A reused)
  int tma3d;               // 2-CTA K-major operands as 3D maps (byte-in-atom, row, atom): bit 0 A, bit 1 B
  const float* bias;       // optional per-output-column bias (OUT_BF16 / OUT_F32): y = fl(acc * scale) + bias
  const __nv_bfloat16* resid;  // OUT_BF16_RESID: residual [M x N] (row stride ld_resid) added in the epilogue
  int64_t ld_resid;
};

// Column bias for the epilogue: 0 outside D or without a bias (warp-uniform address: one
// broadcast load per column, served from L1 after the first tile).
__device__ __forceinline__ float col_bias(const Params& p, int col) {
  return (p.bias != nullptr && col < p.N) ? __ldg(p.bias + col) : 0.0f;
}

// Work unit -> (m0, n0, [kb0, kb1)).
__device__ __forceinline__ void unit_coords(const Params& p, int u, int k_blocks, int& m0, int& n0, int& kb0, int& kb1) {
  const int t = u / p.splits, s = u - t * p.splits;
  m0 = (p.m_fast ? t % p.tiles_m : t / p.tiles_n) * BM;
  n0 = (p.m_fast ? t / p.tiles_m : t % p.tiles_n) * BN;
  kb0 = static_cast<int>((static_cast<int64_t>(k_blocks) * s) / p.splits);
  kb1 = static_cast<int>((static_cast<int64_t>(k_blocks) * (s + 1)) / p.splits);
}

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

#ifdef SB_GEMM_PROBE
// Pipeline probe (tools/gemm_probe.cu only): per CTA {MMA waits on full, MMA waits on tempty,
// MMA-loop cycles, producer waits on empty, epilogue waits on tfull, k-blocks}.
extern __device__ unsigned long long g_probe[1024 * 6];  // defined in build/probe/probe_glue.cu
extern __device__ long long g_trace[4096];               // CTA-pair 0 timeline (globaltimer ns)
extern __device__ unsigned long long g_probe_ns[1024];   // per CTA: MMA-loop wall time (ns), for the clock
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SB_PROBE_T0() const long long sb_t0_ = clock64()
#define SB_PROBE_ADD(slot) atomicAdd(&g_probe[blockIdx.x * 6 + (slot)], (unsigned long long)(clock64() - sb_t0_))
#else
#define SB_PROBE_T0()
#define SB_PROBE_ADD(slot)
#endif

// float(acc) for an s32 accumulator (the epilogue's int8 dequant input). Default: I2F.F32.S32
// (XU pipe). Built with -DSB_I2F_FMA: the same correctly rounded value on the FMA / ALU pipes
// (acc = hi 2^16 + lo, both halves exact in fp32 via the 2^23 magic number, one FMA rounding
// hi 2^16 + lo once; checked against (float)acc on the host for every |acc| < 1e8 and a stride
// beyond). ncu shows the XU pipe ~80% busy in the K = 1280 GEMMs, but the 6-instruction form
// measured slower in the C2 step (fc1 fwd 303 -> 330 us): issue slots, not XU, pace it.
__device__ __forceinline__ float i2f_exact(uint32_t acc) {
#ifndef SB_I2F_FMA
  return static_cast<float>(static_cast<int32_t>(acc));
#else
  const float lo = __fsub_rn(__uint_as_float((acc & 0xffffu) | 0x4b000000u), 8388608.0f);  // 2^23 + lo - 2^23
  const float hi = __fsub_rn(__int_as_float((static_cast<int32_t>(acc) >> 16) + 0x4b400000), 12582912.0f);
  return __fmaf_rn(hi, 65536.0f, lo);
#endif
}

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

__device__ __forceinline__ void epi_bar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory"); }

// Write 8 x 16-byte chunks (one 128-byte row) of this lane into a SW128-swizzled staging row.
__device__ __forceinline__ void stage_row128(uint8_t* buf, int lane, const uint32_t (&w)[32]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int pj = j ^ (lane & 7);
    *reinterpret_cast<uint4*>(buf + lane * 128 + pj * 16) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
  }
}

// Optional L2 evict-first hint on the bf16 output stores (to keep operand tiles resident):
// measured neutral on the C2 int8 GEMMs (302 vs 301 us), so off by default.
#ifndef SB_STORE_EVICT_FIRST
#define SB_STORE_EVICT_FIRST 0
#endif
constexpr bool kStoreEvictFirst = SB_STORE_EVICT_FIRST != 0;

// Arrive on the cluster leader's copy of a barrier (the same smem offset in CTA rank 0).
__device__ __forceinline__ void arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(sbptx::smem_u32(bar) & 0xFEFFFFFFu)
               : "memory");
}

// OUT_BF16_RESID: the warp's 32 x 64 residual tile of a column pair, fetched into registers with
// coalesced 16-byte loads (8 lanes per 128-byte row) one step ahead of its use — pair 0's by the
// caller before it waits for the accumulator, pair 1's right after pair 0's is staged — so the
// HBM latency overlaps the MMAs, the TMEM drain and the previous store instead of stalling the
// epilogue (and, through TMEM, the MMAs).
__device__ __forceinline__ void resid_fetch_pair(const Params& p, uint4 (&rv)[8], int rm0, int ew, int lane, int c0) {
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int rr = t * 4 + (lane >> 3), c = lane & 7;
    const int64_t grow = static_cast<int64_t>(rm0) + ew * 32 + rr;
    rv[t] = make_uint4(0, 0, 0, 0);
    if (grow < p.M && c0 + 8 * c < p.N)
      rv[t] = __ldg(reinterpret_cast<const uint4*>(p.resid + grow * p.ld_resid + c0 + 8 * c));
  }
}

// Drain this CTA's 128 x 256 accumulator (TMEM lane quarter `ew`, column half `half`) to D:
// tcgen05.ld -> scale / convert in registers -> SW128 smem staging -> TMA store (or reduce-add).
// Rows [rm0, rm0 + 128) of D; the TMEM buffer is handed back (`tempty`, on the leader CTA's
// barrier when TWO) as soon as it is drained into registers.
template <int KIND, int OUT, bool SB_COL, bool TWO>
__device__ __forceinline__ void epilogue_tile(const Params& p, const CUtensorMap* tmD, uint32_t t_row, uint64_t* tempty,
                                              int rm0, int n0, int ew, int half, int lane, uint8_t* buf, const float* cs,
                                              float fr, double sa_d, float sb_tensor, uint4 (&rv)[8]) {
  auto resid_fetch = [&](int c0) { resid_fetch_pair(p, rv, rm0, ew, lane, c0); };
#pragma unroll 1
  for (int pr = 0; pr < 2; ++pr) {  // two 64-column pairs per warp
    uint32_t r0[32], r1[32];
#ifdef SB_PROBE_SKIP_LD  // experiment only (tools/gemm_probe): epilogue without the TMEM drain
    for (int j = 0; j < 32; ++j) r0[j] = r1[j] = t_row + j;
#else
    sbptx::tmem_ld_32x32b_x32(t_row + pr * 64, r0);
    sbptx::tmem_ld_32x32b_x32(t_row + pr * 64 + 32, r1);
    sbptx::tmem_ld_wait();
#endif
    if (pr == 1) {
      // accumulator fully drained into registers: hand TMEM back to the MMA warp
      sbptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (TWO)
          arrive_leader(tempty);
        else
          sbptx::mbar_arrive(tempty);
      }
    }
    const int cl = half * 128 + pr * 64;  // column within tile
    const int col0 = n0 + cl;
    if (col0 >= p.N || rm0 >= p.M) continue;  // whole pair outside D (warp-uniform)
    if (OUT == OUT_BF16 || OUT == OUT_BF16_RESID) {
      uint32_t w[32];
      if (OUT == OUT_BF16_RESID) {
        // stage the prefetched residual tile in buf in the SW128 layout stage_row128 uses; each
        // lane then reads its own row
        if (lane == 0) sbptx::tma_store_wait_read<0>();  // previous store done reading buf
        __syncwarp();
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int rr = t * 4 + (lane >> 3), c = lane & 7;
          *reinterpret_cast<uint4*>(buf + rr * 128 + ((c ^ (rr & 7)) * 16)) = rv[t];
        }
        __syncwarp();
        if (pr == 0 && col0 + 64 < p.N) resid_fetch(col0 + 64);  // the next pair's tile
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float a0, a1, b0, b1;
        if (KIND == KIND_I8) {
          a0 = i2f_exact(r0[2 * j]);
          a1 = i2f_exact(r0[2 * j + 1]);
          b0 = i2f_exact(r1[2 * j]);
          b1 = i2f_exact(r1[2 * j + 1]);
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
        if (p.bias != nullptr) {  // fused bias add before the single bf16 rounding
          a0 = __fadd_rn(a0, col_bias(p, col0 + 2 * j));
          a1 = __fadd_rn(a1, col_bias(p, col0 + 2 * j + 1));
          b0 = __fadd_rn(b0, col_bias(p, col0 + 32 + 2 * j));
          b1 = __fadd_rn(b1, col_bias(p, col0 + 32 + 2 * j + 1));
        }
        if (OUT == OUT_BF16_RESID) {  // residual added before the single rounding
          // columns 2j, 2j+1 live in chunk j/4 (a) and 4 + j/4 (b) of this lane's staged row
          const uint32_t ra = *reinterpret_cast<const uint32_t*>(buf + lane * 128 + (((j >> 2) ^ (lane & 7)) * 16) +
                                                                 (j & 3) * 4);
          const uint32_t rb = *reinterpret_cast<const uint32_t*>(
              buf + lane * 128 + (((4 + (j >> 2)) ^ (lane & 7)) * 16) + (j & 3) * 4);
          const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ra));
          const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&rb));
          a0 = __fadd_rn(a0, fa.x);
          a1 = __fadd_rn(a1, fa.y);
          b0 = __fadd_rn(b0, fb.x);
          b1 = __fadd_rn(b1, fb.y);
        }
        w[j] = pack_bf16x2(a0, a1);
        w[16 + j] = pack_bf16x2(b0, b1);
      }
#ifdef SB_PROBE_SKIP_STORE  // experiment only (tools/gemm_probe): no output staging / TMA store
      if (w[0] == 0x7fc00001u) buf[0] = 0;  // keep the math live
      continue;
#endif
      if (OUT != OUT_BF16_RESID) {
        if (lane == 0) sbptx::tma_store_wait_read<0>();  // previous store done reading buf
      }
      __syncwarp();  // (RESID: every lane has read its residual row before buf is overwritten)
      stage_row128(buf, lane, w);  // 64 bf16 = 128 B per row
      sbptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (kStoreEvictFirst)
          sbptx::tma_store_2d_hint(tmD, buf, col0, rm0 + ew * 32, sbptx::l2_policy_evict_first());
        else
          sbptx::tma_store_2d(tmD, buf, col0, rm0 + ew * 32);
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
            const float v = KIND == KIND_I8 ? i2f_exact(r[j]) : __uint_as_float(r[j]);
            const float y = SB_COL ? __fmul_rn(v, fr * cs[cc + j]) : __fmul_rn(v, fr);
            // bias as a separate rounded add: identical bits to an unfused y + bias
            w[j] = __float_as_uint(p.bias != nullptr ? __fadd_rn(y, col_bias(p, n0 + cc + j)) : y);
          }
        }
        if (lane == 0) sbptx::tma_store_wait_read<0>();
        __syncwarp();
        stage_row128(buf, lane, w);  // 32 x 4 B = 128 B per row
        sbptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (OUT == OUT_F32_RAW_ADD) {
            asm volatile(
                "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(tmD)),
                "r"(sbptx::smem_u32(buf)), "r"(n0 + cc), "r"(rm0 + ew * 32)
                : "memory");
          } else {
            sbptx::tma_store_2d(tmD, buf, n0 + cc, rm0 + ew * 32);
          }
          sbptx::tma_store_commit();
        }
      }
    }
  }
}

template <int KIND, bool A_MN, bool B_MN, int OUT, bool SB_COL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmD, const Params p, uint32_t idesc_runtime) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + STAGES * A_STAGE_BYTES;
  uint8_t* smem_epi = smem + STAGES * STAGE_BYTES;
  float* col_scale = reinterpret_cast<float*>(smem_epi + EPI_WARPS * EPI_BUF_BYTES);  // [BN]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(col_scale + BN);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_tiles = p.tiles_m * p.tiles_n * p.splits;  // work units
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
      sbptx::mbar_init(&tempty_bar[a], EPI_WARPS);
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
        int m0, n0, kb0, kb1;
        unit_coords(p, t, k_blocks, m0, n0, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            SB_PROBE_T0();
            sbptx::mbar_wait(&empty_bar[stage], phase ^ 1u);
            SB_PROBE_ADD(3);
          }
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
#ifdef SB_GEMM_PROBE
      const long long sb_loop0 = clock64();
#endif
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        {
          SB_PROBE_T0();
          sbptx::mbar_wait(&tempty_bar[acc], acc_phase ^ 1u);
          SB_PROBE_ADD(1);
        }
        sbptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        int m0_, n0_, kb0, kb1;
        unit_coords(p, t, k_blocks, m0_, n0_, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            SB_PROBE_T0();
            sbptx::mbar_wait(&full_bar[stage], phase);
            SB_PROBE_ADD(0);
          }
#ifdef SB_GEMM_PROBE
          atomicAdd(&g_probe[blockIdx.x * 6 + 5], 1ull);
#endif
          sbptx::tc_fence_after();
          const uint32_t a_addr = sbptx::smem_u32(smem_a + stage * A_STAGE_BYTES);
          const uint32_t b_addr = sbptx::smem_u32(smem_b + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = operand_desc<A_MN>(a_addr, k);
            const uint64_t bd = operand_desc<B_MN>(b_addr, k);
            if (KIND == KIND_I8)
              sbptx::mma_i8(d_tmem, ad, bd, idesc, (kb != kb0) || k);
            else if (KIND == KIND_F8)
              sbptx::mma_f8(d_tmem, ad, bd, idesc, (kb != kb0) || k);
            else
              sbptx::mma_f16(d_tmem, ad, bd, idesc, (kb != kb0) || k);
          }
          sbptx::mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        sbptx::mma_commit(&tfull_bar[acc]);
      }
#ifdef SB_GEMM_PROBE
      atomicAdd(&g_probe[blockIdx.x * 6 + 2], (unsigned long long)(clock64() - sb_loop0));
#endif
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    constexpr bool SCALED = OUT == OUT_BF16 || OUT == OUT_BF16_RESID || OUT == OUT_F32 || OUT == OUT_F32_EXACT;
    const int ew = warp & 3;               // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;      // column half of the tile
    const int ei = threadIdx.x - 128;      // 0..255 within the epilogue group
    uint8_t* buf = smem_epi + (warp - 4) * EPI_BUF_BYTES;
    const float sb_tensor = (SCALED && !SB_COL) ? __ldg(p.sb) : 1.0f;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      int m0, n0, kb0_, kb1_;
      unit_coords(p, t, k_blocks, m0, n0, kb0_, kb1_);
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      float* cs = col_scale;  // single buffer: the first barrier below orders reuse
      if (SCALED && SB_COL) {
        // stage this tile's per-column states once (all 8 epilogue warps, 256 threads)
        epi_bar_sync();
        cs[ei] = (n0 + ei) < p.N ? __ldg(p.sb + n0 + ei) : 0.0f;
        epi_bar_sync();
      }
      const int row = m0 + ew * 32 + lane;
      float fr = 1.0f;       // per-row factor: sa_i * post (* sb for a tensor-wise B)
      double sa_d = 1.0;
      if (SCALED) {
        const float s = row < p.M ? __ldg(p.sa + (p.sa_stride ? row : 0)) : 0.0f;
        sa_d = static_cast<double>(s);
        fr = SB_COL ? s * p.post_scale : s * p.post_scale * sb_tensor;
      }
      uint4 rv[8];
      if (OUT == OUT_BF16_RESID && m0 < p.M) resid_fetch_pair(p, rv, m0, ew, lane, n0 + half * 128);
      {
        SB_PROBE_T0();
        sbptx::mbar_wait(&tfull_bar[acc], acc_phase);
        if (lane == 0 && warp == 4) SB_PROBE_ADD(4);
      }
      sbptx::tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + half * 128;
      epilogue_tile<KIND, OUT, SB_COL, false>(p, &tmD, t_row, &tempty_bar[acc], m0, n0, ew, half, lane, buf, cs, fr,
                                             sa_d, sb_tensor, rv);
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
