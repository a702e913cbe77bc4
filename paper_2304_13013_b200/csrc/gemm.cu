// gemm.cu — host launchers for the SwitchBack GEMMs plus their exact / SIMT companions.
//
//   sb::gemm_i8    int8_matmul_dequant / matmul_dequant_dual_rowwise (linear.cpp:39-83)
//                  tcgen05 kind::i8 when the operands are TMA-legal (K % 16 == 0, 16-B
//                  aligned, K <= 133144 so s32 cannot overflow); otherwise a SIMT kernel
//                  with int64 accumulation (the reference's own int64 switch, linear.cpp:62-65).
//   sb::wgrad      wgrad_full_precision (linear.cpp:193-195): tcgen05 kind::f16 over MN-major
//                  bf16 G and X, or the exact sequential fp32 kernel (matrix.cpp:53-68).
//   sb::matmul_f32_seq  matmul (matrix.cpp:53-68): one output per thread, strictly sequential
//                  fp32 sum with separately rounded multiply and add (-ffp-contract=off).
//   sb::gemm_fp8   fp8 SwitchBack GEMM (tcgen05 kind::f8f6f4).
#include <cuda_bf16.h>

#include <mutex>

#include "sb_internal.h"
#include "tc_gemm.cuh"
#include "tc_gemm2.cuh"
#include "tc_dw_wide.cuh"
#include "tc_i8_wide.cuh"

#include <cstdio>
#include <cstdlib>

namespace {

constexpr int64_t kInt32SafeInner = 2147483647LL / (127 * 127);  // 133144, linear.cpp:37

// ----------------------------------------------------------- SIMT int8 ----
// Fallback for operands the TMA path cannot take (K % 16 != 0, unaligned rows) and for
// K > 133144, where the reference switches to an int64 accumulator (linear.cpp:62-65).
// 64 x 64 outputs per block, 4 x 4 per thread; K tiles of 64 bytes staged in smem as packed
// 4-byte words so each step is one dp4a per output. A tile's partial sum is at most
// 64 * 127^2 < 2^31 in int32; tiles accumulate in int64, so the result is the exact integer
// product for any K. Rows go on grid.y in steps of gridDim.y (no 65535-row limit).
constexpr int kSimtTile = 64, kSimtKw = 16;  // 16 words = 64 bytes of K per tile

__device__ __forceinline__ int load_word(const int8_t* __restrict__ row, int64_t k, int64_t K) {
  uint32_t v = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (k + b < K) v |= static_cast<uint32_t>(static_cast<uint8_t>(row[k + b])) << (8 * b);
  return static_cast<int>(v);
}

template <int OUT>
__global__ void __launch_bounds__(256) k_gemm_i8_simt(const int8_t* __restrict__ qa, const float* __restrict__ sa,
                                                      int sa_stride, const int8_t* __restrict__ qb,
                                                      const float* __restrict__ sb, int sb_stride, int64_t M,
                                                      int64_t N, int64_t K, void* __restrict__ out) {
  __shared__ int As[kSimtKw][kSimtTile + 1];
  __shared__ int Bs[kSimtKw][kSimtTile + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kSimtTile;
  for (int64_t i0 = static_cast<int64_t>(blockIdx.y) * kSimtTile; i0 < M; i0 += static_cast<int64_t>(gridDim.y) * kSimtTile) {
    int64_t acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = 0;
    for (int64_t k0 = 0; k0 < K; k0 += 4 * kSimtKw) {
      for (int e = threadIdx.x; e < kSimtKw * kSimtTile; e += 256) {
        const int kw = e / kSimtTile, rr = e % kSimtTile;
        const int64_t ia = i0 + rr, jb = j0 + rr, kg = k0 + 4 * kw;
        As[kw][rr] = (ia < M && kg < K) ? load_word(qa + ia * K, kg, K) : 0;
        Bs[kw][rr] = (jb < N && kg < K) ? load_word(qb + jb * K, kg, K) : 0;
      }
      __syncthreads();
      int part[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) part[u][v] = 0;
#pragma unroll 4
      for (int kw = 0; kw < kSimtKw; ++kw) {
        int av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = As[kw][ty * 4 + u];
#pragma unroll
        for (int v = 0; v < 4; ++v) bv[v] = Bs[kw][tx * 4 + v];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) part[u][v] = __dp4a(av[u], bv[v], part[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] += part[u][v];
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + ty * 4 + u;
      if (i >= M) continue;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int64_t j = j0 + tx * 4 + v;
        if (j >= N) continue;
        const int64_t o = i * N + j;
        const int64_t a = acc[u][v];
        if (OUT == 5) {  // raw int64
          static_cast<int64_t*>(out)[o] = a;
        } else if (OUT == sbtc::OUT_I32) {
          static_cast<int32_t*>(out)[o] = static_cast<int32_t>(a);
        } else {
          const float si = sa[sa_stride ? i : 0], sj = sb[sb_stride ? j : 0];
          if (OUT == sbtc::OUT_F32_EXACT)  // linear.cpp:49, left to right in double
            static_cast<float*>(out)[o] = __double2float_rn(
                __ddiv_rn(__dmul_rn(__dmul_rn(static_cast<double>(a), static_cast<double>(si)), static_cast<double>(sj)),
                          16129.0));
          else if (OUT == sbtc::OUT_F32)
            static_cast<float*>(out)[o] = static_cast<float>(a) * (si / 16129.0f) * sj;
          else
            static_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(static_cast<float>(a) * (si / 16129.0f) * sj);
        }
      }
    }
  }
}

// --------------------------------------------------- exact sequential fp32 ----
// y[i][j] (+)= sum_p a(i,p) * b(j,p), p ascending, fmul/fadd separately rounded.
// 64 x 64 outputs per block, 4 x 4 per thread, k-tiles of 16 staged in smem.
__device__ __forceinline__ void store_out(float* p, float v) { *p = v; }
__device__ __forceinline__ void store_out(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ float load_out(const float* p) { return *p; }
__device__ __forceinline__ float load_out(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T, typename TO = float>
__global__ void __launch_bounds__(256) k_matmul_seq(const T* __restrict__ a, int64_t a_rs, int64_t a_ks,
                                                    const T* __restrict__ b, int64_t b_rs, int64_t b_ks, int64_t R,
                                                    int64_t Cc, int64_t K, TO* __restrict__ y, int accumulate) {
  __shared__ float As[16][64 + 1];
  __shared__ float Bs[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 64, j0 = static_cast<int64_t>(blockIdx.x) * 64;
  float acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0f;
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, rr = e % 64;
      const int64_t ia = i0 + rr, jb = j0 + rr, kg = k0 + kk;
      As[kk][rr] = (ia < R && kg < K) ? static_cast<float>(a[ia * a_rs + kg * a_ks]) : 0.0f;
      Bs[kk][rr] = (jb < Cc && kg < K) ? static_cast<float>(b[jb * b_rs + kg * b_ks]) : 0.0f;
    }
    __syncthreads();
    const int kmax = static_cast<int>(K - k0 < 16 ? K - k0 : 16);
    for (int kk = 0; kk < kmax; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[kk][ty * 4 + u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = Bs[kk][tx * 4 + v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = __fadd_rn(acc[u][v], __fmul_rn(av[u], bv[v]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t i = i0 + ty * 4 + u, j = j0 + tx * 4 + v;
      if (i < R && j < Cc) store_out(y + i * Cc + j, accumulate ? __fadd_rn(load_out(y + i * Cc + j), acc[u][v]) : acc[u][v]);
    }
}

// -------------------------------------------------------------- SIMT fp8 ----
__device__ __forceinline__ float dec_fp8(uint8_t b, int fmt) {
  const uint32_t s = (b >> 7) & 1u;
  float v;
  if (fmt == 0) {
    const uint32_t e = (b >> 3) & 0xFu, m = b & 7u;
    v = e == 0 ? ldexpf(static_cast<float>(m), -9) : ldexpf(1.0f + m / 8.0f, static_cast<int>(e) - 7);
  } else {
    const uint32_t e = (b >> 2) & 0x1Fu, m = b & 3u;
    v = e == 0 ? ldexpf(static_cast<float>(m), -16) : ldexpf(1.0f + m / 4.0f, static_cast<int>(e) - 15);
  }
  return s ? -v : v;
}

__global__ void k_gemm_fp8_simt(const uint8_t* __restrict__ qa, int fa, const float* __restrict__ sa, int sa_stride,
                                const uint8_t* __restrict__ qb, int fb, const float* __restrict__ sb, int sb_stride,
                                int64_t M, int64_t N, int64_t K, void* __restrict__ out, int out_bf16) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= N) return;
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y) {  // no 65535-row grid limit
    float acc = 0.0f;
    for (int64_t p = 0; p < K; ++p) acc = fmaf(dec_fp8(qa[i * K + p], fa), dec_fp8(qb[j * K + p], fb), acc);
    const float y = acc * sa[sa_stride ? i : 0] * sb[sb_stride ? j : 0];
    if (out_bf16)
      static_cast<__nv_bfloat16*>(out)[i * N + j] = __float2bfloat16_rn(y);
    else
      static_cast<float*>(out)[i * N + j] = y;
  }
}

// ------------------------------------------------------------ TMA maps ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// A GEMM operand as a 2-D row-major global tensor: `inner` contiguous elements per row,
// `outer` rows. mn = the operand is MN-major (its contiguous dimension is M or N).
struct Operand {
  const void* ptr;
  CUtensorMapDataType dt;
  uint64_t inner, outer, stride_bytes;
  bool mn;
  uint32_t kbox;  // K-major: elements per 128-byte K slice (128 for 8-bit, 64 for bf16)
};

// K-major operand as a 3D map (element-in-atom, row, atom) with box {kbox, rows, atoms}: one TMA
// per stage per operand in the 2-CTA kernel. False when K is not a whole number of atoms.
bool encode_operand3d(CUtensorMap* m, const Operand& o, uint32_t rows, uint32_t atoms) {
  if (o.mn || o.inner % o.kbox != 0) return false;
  EncodeFn fn = get_encode();
  if (!fn) return false;
  const cuuint64_t dims[3] = {o.kbox, o.outer, o.inner / o.kbox};
  const cuuint64_t strides[2] = {o.stride_bytes, 128};
  const cuuint32_t box[3] = {o.kbox, rows, atoms};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, o.dt, 3, const_cast<void*>(o.ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// SB_TMA3D=1 loads the 2-CTA GEMM's K-major operands with one 3D TMA per stage (measured neutral on
// the C2 step, 2.75 vs 2.75 ms: the producer is not the bottleneck there; default off).
bool tma3d_enabled() {
  static int v = -1;
  if (v < 0) v = getenv("SB_TMA3D") ? atoi(getenv("SB_TMA3D")) : 0;
  return v != 0;
}

// rows: box rows of a K-major operand; mn_krows: k-rows per box of an MN-major one.
bool encode_operand(CUtensorMap* m, const Operand& o, uint32_t rows, uint32_t mn_krows) {
  if (o.mn)
    return sb::encode_tmap_2d(m, o.dt, o.ptr, o.inner, o.outer, o.stride_bytes, 64, mn_krows, CU_TENSOR_MAP_SWIZZLE_128B);
  return sb::encode_tmap_2d(m, o.dt, o.ptr, o.inner, o.outer, o.stride_bytes, o.kbox, rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

// 2-CTA (cta_group::2, 256 x 256 tiles, tc_gemm2.cuh) whenever the problem has at least one
// 256-row tile per SM pair's worth of work; 1-CTA 128 x 256 (tc_gemm.cuh) for small M.
// SB_GEMM_2CTA=0/1 in the environment overrides the AUTO choice; sb_set_gemm_path overrides both.
bool use_2cta(sb_handle h, int64_t M, int64_t units256) {
  if (h->gemm_path == SB_GEMM_1CTA || h->num_sms < 2) return false;
  if (h->gemm_path == SB_GEMM_2CTA || h->gemm_path == SB_GEMM_2CTA_MC) return true;
  static int env = -2;
  if (env == -2) {
    const char* e = getenv("SB_GEMM_2CTA");
    env = e ? (e[0] == '1' ? 1 : 0) : -1;
  }
  if (env >= 0) return env == 1;
  return M > 128 && units256 >= h->num_sms / 2;
}

// Per-device cache of a cluster kernel's one-time setup (the max-dynamic-smem attribute is per
// device context, and so is the co-resident cluster count).
struct PairCache {
  std::once_flag once[16];
  cudaError_t err[16] = {};
  int pairs[16] = {};
};
template <typename Kern>
int cluster_pairs(sb_handle h, PairCache& c, Kern kern, int smem, int threads, cudaError_t* err, int csize = 2) {
  const int d = h->device & 15;
  std::call_once(c.once[d], [&] {
    c.err[d] = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize * (h->num_sms / csize));
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = csize;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (c.err[d] != cudaSuccess || cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1)
      n = h->num_sms / csize;
    c.pairs[d] = n;
    cudaGetLastError();
  });
  *err = c.err[d];
  return c.pairs[d];
}

// 2-CTA launch of pipeline shape CFG (tc_gemm2.cuh Pipe2); `units` = pair tiles (CFG 0 / 1)
// or cluster-of-4 units (CFG 2). Persistent grid: only as many clusters as can be co-resident
// (a pair needs two SMs of one TPC); launching more would run the surplus as a second wave.
template <int KIND, int OUT, bool A_MN, bool B_MN, bool SB_COL, int CFG>
cudaError_t launch_2cta_cfg(sb_handle h, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& d,
                            const sbtc::Params& p, uint32_t idesc, int units) {
  auto kern = sbtc2::k_tc_gemm2<KIND, A_MN, B_MN, OUT, SB_COL, CFG>;
  constexpr int CL = sbtc2::Pipe2<CFG>::CL;
  static PairCache cache;
  cudaError_t err = cudaSuccess;
  const int max_clusters = cluster_pairs(h, cache, kern, sbtc2::SMEM2_BYTES, sbtc::NUM_THREADS, &err, CL);
  if (err != cudaSuccess) return err;
  if (getenv("SB_DEBUG")) fprintf(stderr, "[sb] 2-CTA GEMM (cfg %d): %d co-resident clusters of %d\n", CFG, max_clusters, CL);
  const int grid = CL * (units < max_clusters ? units : max_clusters);
  sb::launch_pdl(kern, dim3(grid), dim3(sbtc::NUM_THREADS), sbtc2::SMEM2_BYTES, h->stream, ta, tb, d, p, idesc);
  return cudaGetLastError();
}

// SB_GEMM_CFG=0|1|2 picks the 2-CTA pipeline shape (tc_gemm2.cuh Pipe2; default 0).
int gemm2_cfg() {
  static int c = -1;
  if (c < 0) c = getenv("SB_GEMM_CFG") ? atoi(getenv("SB_GEMM_CFG")) : 0;
  return c;
}
// Pipeline shape for one 2-CTA launch: SB_GEMM_2CTA_MC forces the cluster-of-4 multicast form,
// SB_GEMM_CFG in the environment overrides AUTO, and AUTO takes the multicast form for the
// 8-bit GEMMs when there is at least one cluster unit per co-resident cluster.
int gemm2_cfg_for(sb_handle h, const sbtc::Params& p) {
  if (h->gemm_path == SB_GEMM_2CTA_MC) return 2;
  if (getenv("SB_GEMM_CFG")) return gemm2_cfg();
  (void)p;
  return 0;
}
constexpr int kCfgMnKrows[3] = {64 * sbtc2::Pipe2<0>::ATOMS, 64 * sbtc2::Pipe2<1>::ATOMS, 64 * sbtc2::Pipe2<2>::ATOMS};

template <int KIND, int OUT, bool A_MN, bool B_MN, bool SB_COL>
cudaError_t launch_2cta(sb_handle h, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& d,
                        const sbtc::Params& p, uint32_t idesc, int units, int cfg) {
  if (cfg == 1) return launch_2cta_cfg<KIND, OUT, A_MN, B_MN, SB_COL, 1>(h, ta, tb, d, p, idesc, units);
  if (cfg == 2) {
    const int units4 = ((p.tiles_m + 1) / 2) * p.tiles_n * p.splits;
    return launch_2cta_cfg<KIND, OUT, A_MN, B_MN, SB_COL, 2>(h, ta, tb, d, p, idesc, units4);
  }
  return launch_2cta_cfg<KIND, OUT, A_MN, B_MN, SB_COL, 0>(h, ta, tb, d, p, idesc, units);
}

template <int KIND, int OUT, bool A_MN = false, bool B_MN = false, bool SB_COL = false>
cudaError_t launch_tc(sb_handle h, const Operand& A, const Operand& B, const CUtensorMap& d, sbtc::Params p,
                      uint32_t idesc) {
  const int64_t units256 = ((p.M + 255) / 256) * ((p.N + sbtc::BN - 1) / sbtc::BN) * (p.splits < 1 ? 1 : p.splits);
  const bool two = use_2cta(h, p.M, units256);
  CUtensorMap ta, tb;
  const int cfg = two ? gemm2_cfg_for(h, p) : 0;
  const int mnk = two ? kCfgMnKrows[cfg] : 64;
  if (!encode_operand(&ta, A, 128, mnk) || !encode_operand(&tb, B, two ? 128 : 256, mnk))
    return cudaErrorInvalidValue;
  p.tma3d = 0;
  if (two && tma3d_enabled()) {
    const int atoms = cfg == 1 ? sbtc2::Pipe2<1>::ATOMS : sbtc2::Pipe2<0>::ATOMS;
    CUtensorMap t3;
    if (!A.mn && encode_operand3d(&t3, A, 128, atoms)) {
      ta = t3;
      p.tma3d |= 1;
    }
    if (!B.mn && encode_operand3d(&t3, B, 128, atoms)) {
      if (cfg != 2) {  // the cluster-of-4 form multicasts B atom by atom (2D boxes)
        tb = t3;
        p.tma3d |= 2;
      }
    }
  }
  p.tiles_m = static_cast<int>((p.M + (two ? sbtc2::BM2 : sbtc::BM) - 1) / (two ? sbtc2::BM2 : sbtc::BM));
  p.tiles_n = static_cast<int>((p.N + sbtc::BN - 1) / sbtc::BN);
  if (p.splits < 1) p.splits = 1;
  const int units = p.tiles_m * p.tiles_n * p.splits;
  h->launches++;
  if (two) return launch_2cta<KIND, OUT, A_MN, B_MN, SB_COL>(h, ta, tb, d, p, idesc, units, cfg);
  // the max-dynamic-smem attribute is per device context: set once per device
  static std::once_flag once1[16];
  static cudaError_t attr_err1[16] = {};
  const int dv = h->device & 15;
  std::call_once(once1[dv], [dv] {
    attr_err1[dv] = cudaFuncSetAttribute(sbtc::k_tc_gemm<KIND, A_MN, B_MN, OUT, SB_COL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, sbtc::SMEM_BYTES);
  });
  if (attr_err1[dv] != cudaSuccess) return attr_err1[dv];
  const int grid = units < h->num_sms ? units : h->num_sms;
  sbtc::k_tc_gemm<KIND, A_MN, B_MN, OUT, SB_COL><<<grid, sbtc::NUM_THREADS, sbtc::SMEM_BYTES, h->stream>>>(
      ta, tb, d, p, idesc);
  return cudaGetLastError();
}

// One-wave 256 x 384 dW (tc_dw_wide.cuh) when one orientation fits the SM pairs in a single
// wave; cudaErrorNotSupported = use the 256 x 256 split-K path. G: A operand (MN-major, m
// wide), X: B operand (n wide); TRANS runs C = X^T G and stores C^T.
// rq (optional): also quantize G row-wise inside the same launch (tc_dw_wide.cuh QV).
// Co-resident pairs of the one-wave dW kernel on h's device (its smem attributes set once per
// device context); <= 0 when the kernel is off (SB_DW_WIDE=0, 1-CTA path) or cannot launch.
int dw_wide_pairs(sb_handle h) {
  static int env = -1;
  if (env < 0) env = getenv("SB_DW_WIDE") ? atoi(getenv("SB_DW_WIDE")) : 1;
  if (!env || h->gemm_path == SB_GEMM_1CTA || h->num_sms < 2) return 0;
  static int max_pairs_d[16] = {};
  static cudaError_t attr_err_d[16] = {};
  static std::once_flag once_d[16];
  const int dv = h->device & 15;
  int& max_pairs = max_pairs_d[dv];
  cudaError_t& attr_err = attr_err_d[dv];
  std::call_once(once_d[dv], [&] {
    for (auto kern : {sbdw::k_dw_wide<false, 0>, sbdw::k_dw_wide<true, 0>, sbdw::k_dw_wide<false, sbdw::kQV>,
                      sbdw::k_dw_wide<true, sbdw::kQV>}) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sbdw::SMEM_BYTES);
      if (e != cudaSuccess) attr_err = e;
    }
    for (auto kern : {sbdw::k_dw_wide<false, 0, 8>, sbdw::k_dw_wide<true, 0, 8>, sbdw::k_dw_wide<false, sbdw::kQV, 8>,
                      sbdw::k_dw_wide<true, sbdw::kQV, 8>}) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sbdw::SMEM_BYTES);
      if (e != cudaSuccess) attr_err = e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * (h->num_sms / 2));
    cfg.blockDim = dim3(sbtc::NUM_THREADS);
    cfg.dynamicSmemBytes = sbdw::SMEM_BYTES;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n_ = 0;
    if (attr_err != cudaSuccess || cudaOccupancyMaxActiveClusters(&n_, sbdw::k_dw_wide<false, 0>, &cfg) != cudaSuccess ||
        n_ < 1)
      n_ = h->num_sms / 2;
    max_pairs = n_;
    cudaGetLastError();
  });
  return attr_err != cudaSuccess ? 0 : max_pairs;
}

// The one-wave dW tiling plan for an m x n dW on max_pairs co-resident pairs: false = use the
// 256 x 256 path. Both orientations are tried; with one wave in either, the one with fewer tiles
// (e.g. 3840 x 1280: 50 full 256 x 384 tiles transposed against 60 with 15 of them a third wide,
// 489 vs 510 us). Worth it only when the 256 x 256 tiling would leave a partial wave and the
// one-wave tiling keeps most pairs busy.
bool dw_wide_plan(int max_pairs, int64_t m, int64_t n, bool* trans) {
  const int64_t u_direct = ((m + sbdw::WM - 1) / sbdw::WM) * ((n + sbdw::WN - 1) / sbdw::WN);
  const int64_t u_trans = ((n + sbdw::WM - 1) / sbdw::WM) * ((m + sbdw::WN - 1) / sbdw::WN);
  const bool d_ok = u_direct <= max_pairs, t_ok = u_trans <= max_pairs;
  if (!d_ok && !t_ok) return false;
  *trans = !d_ok || (t_ok && u_trans < u_direct);
  const int64_t u256 = ((m + 255) / 256) * ((n + 255) / 256);
  return !(u256 % max_pairs == 0 || std::max(d_ok ? u_direct : 0, t_ok ? u_trans : 0) * 4 < max_pairs * 3);
}

cudaError_t launch_dw_wide(sb_handle h, const Operand& G, const Operand& X, const CUtensorMap& td, int64_t m, int64_t n,
                           int64_t T, const sb::RowQuant* rq, const sbdw::DMaps<8>* rs = nullptr) {
  const int max_pairs = dw_wide_pairs(h);
  if (max_pairs <= 0) return cudaErrorNotSupported;
  bool trans = false;
  if (!dw_wide_plan(max_pairs, m, n, &trans)) return cudaErrorNotSupported;
  const Operand& Aop = trans ? X : G;
  const Operand& Bop = trans ? G : X;
  CUtensorMap ta, tb;
  if (!encode_operand(&ta, Aop, 128, 64) || !encode_operand(&tb, Bop, 128, 64)) return cudaErrorInvalidValue;
  sbdw::WParams p{};
  p.M = static_cast<int>(trans ? n : m);
  p.N = static_cast<int>(trans ? m : n);
  p.K = static_cast<int>(T);
  p.tiles_m = static_cast<int>((p.M + sbdw::WM - 1) / sbdw::WM);
  p.tiles_n = static_cast<int>((p.N + sbdw::WN - 1) / sbdw::WN);
  const int units = p.tiles_m * p.tiles_n;
  int qv = 0;
  if (rq) {
    // G [T x m] row-major bf16 (its MN-major operand view), rows of m / 8 16-byte vectors
    const int nvec = static_cast<int>(m / 8);
    qv = sbdw::kQV;
    p.qg = static_cast<const __nv_bfloat16*>(G.ptr);
    p.q_rows = T;
    p.q_ld = m;
    p.q_nvec = nvec;
    p.q_out = rq->q;
    p.q_ldq = rq->ldq;
    p.q_state = rq->state;
    p.q_err = h->d_err;
    static int qw = -1;  // SB_DWQ_WARPS: quantizing warps per CTA (measurement knob)
    if (qw < 0) qw = getenv("SB_DWQ_WARPS") ? std::max(1, std::min(10, atoi(getenv("SB_DWQ_WARPS")))) : 10;
    p.q_warps = qw;
    static int lag = INT32_MIN;  // SB_DWQ_LAG: pacing distance behind the producer, k-blocks (measurement knob)
    if (lag == INT32_MIN) lag = getenv("SB_DWQ_LAG") ? atoi(getenv("SB_DWQ_LAG")) : sbdw::kLag;
    p.q_lag = lag;
  }
  // with a fused quantize every co-resident pair takes part (pairs without a tile only quantize)
  const int grid = 2 * (rq ? max_pairs : (units < max_pairs ? units : max_pairs));
  if (rq && units < max_pairs) {
    // the tile-less pairs' share of G's k-blocks (SB_DWQ_IDLE: fraction of all k-blocks)
    static double frac = -1.0;
    if (frac < 0) frac = getenv("SB_DWQ_IDLE") ? atof(getenv("SB_DWQ_IDLE")) : 0.0;
    const int64_t qkb = (T + sbdw::KROWS - 1) / sbdw::KROWS;
    p.q_idle_kb = static_cast<int>(std::min<double>(static_cast<double>(qkb), frac * static_cast<double>(qkb)));
  }
  h->launches++;
  if (rs) {
    auto go8 = [&](auto kern) {
      sb::launch_pdl(kern, dim3(grid), dim3(sbtc::NUM_THREADS), sbdw::SMEM_BYTES, h->stream, ta, tb, *rs, p);
    };
    if (qv)
      trans ? go8(sbdw::k_dw_wide<true, sbdw::kQV, 8>) : go8(sbdw::k_dw_wide<false, sbdw::kQV, 8>);
    else
      trans ? go8(sbdw::k_dw_wide<true, 0, 8>) : go8(sbdw::k_dw_wide<false, 0, 8>);
    return cudaGetLastError();
  }
  sbdw::DMaps<1> d1{};
  d1.m[0] = td;
  d1.world = 1;
  d1.nblocks = 1;
  auto go = [&](auto kern) {
    sb::launch_pdl(kern, dim3(grid), dim3(sbtc::NUM_THREADS), sbdw::SMEM_BYTES, h->stream, ta, tb, d1, p);
  };
  if (qv)
    trans ? go(sbdw::k_dw_wide<true, sbdw::kQV>) : go(sbdw::k_dw_wide<false, sbdw::kQV>);
  else
    trans ? go(sbdw::k_dw_wide<true, 0>) : go(sbdw::k_dw_wide<false, 0>);
  return cudaGetLastError();
}

// The 256 x 384 int8 / fp8 kernel runs when forced (sb_set_gemm_path(h, SB_GEMM_WIDE)) or with
// SB_GEMM_WIDE=1 in the environment; AUTO keeps the 256 x 256 kernel, which measured faster at
// the C2 shapes (tools/gemm_probe.cu with the effective-clock readout: 256 x 256 is 95% MMA-busy
// in its main loop at K = 5120 and 76% at K = 1280; 256 x 384 86% / 57%, its 16 epilogue warps
// taking issue slots and shared-memory bandwidth from the MMA / TMA warps).
bool wide_enabled(sb_handle h) {
  static int env = -1;
  if (env < 0) env = getenv("SB_GEMM_WIDE") ? atoi(getenv("SB_GEMM_WIDE")) : 0;
  if (h->gemm_path == SB_GEMM_WIDE) return true;
  return env != 0 && h->gemm_path == SB_GEMM_AUTO && h->num_sms >= 2;
}

// The transposed 256 x 384 GEMM (tc_i8_wide.cuh): D[M x N] = X[M x K] . W[N x K]^T computed as
// W . X^T. W (weight rows) is the MMA's A operand, X (tokens) its B operand. Returns
// cudaErrorNotSupported when the shape is better served by the 256 x 256 kernels (too few
// tiles to fill the SM pairs).
template <int KIND, int OUT, bool SB_COL>
cudaError_t launch_wide_t(sb_handle h, const CUtensorMap& tw, const CUtensorMap& tx, const CUtensorMap& tx2,
                          const CUtensorMap& td, const sbwide::WideParams& p, uint32_t idesc) {
  static PairCache cache;
  auto kern = sbwide::k_gemm_wide<KIND, OUT, SB_COL>;
  cudaError_t err;
  const int pairs = cluster_pairs(h, cache, kern, sbwide::SMEM_BYTES, sbwide::THREADS, &err);
  if (err != cudaSuccess) return err;
  const int units = p.tiles_w * p.tiles_t;
  const int grid = 2 * (units < pairs ? units : pairs);
  h->launches++;
  sb::launch_pdl(kern, dim3(grid), dim3(sbwide::THREADS), sbwide::SMEM_BYTES, h->stream, tw, tx, tx2, td, p, idesc);
  return cudaGetLastError();
}

// w: N x K (weight rows), x: M x K (tokens), both K-major 8-bit; out: M x N (bf16 / f32 / s32).
cudaError_t launch_wide(sb_handle h, int kind, int out_mode, bool sb_col, const void* x, const void* w, int64_t M,
                        int64_t N, int64_t K, const float* sa, const float* sbp, float post, const float* bias,
                        void* out, sb_dtype out_dt, uint32_t idesc) {
  if (!wide_enabled(h)) return cudaErrorNotSupported;
  const int64_t tiles_w = (N + sbwide::TW - 1) / sbwide::TW, tiles_t = (M + sbwide::TT - 1) / sbwide::TT;
  // enough tiles for every SM pair to take several (the last partial wave costs little)
  if (h->gemm_path != SB_GEMM_WIDE && tiles_w * tiles_t < 4 * (h->num_sms / 2)) return cudaErrorNotSupported;
  const CUtensorMapDataType u8 = CU_TENSOR_MAP_DATA_TYPE_UINT8;
  CUtensorMap tw, tx, tx2, td;
  const bool ok =
      sb::encode_tmap_2d(&tw, u8, w, K, N, K, sbwide::KB, 128, CU_TENSOR_MAP_SWIZZLE_128B) &&
      sb::encode_tmap_2d(&tx, u8, x, K, M, K, sbwide::KB, 128, CU_TENSOR_MAP_SWIZZLE_128B) &&
      sb::encode_tmap_2d(&tx2, u8, x, K, M, K, sbwide::KB, 64, CU_TENSOR_MAP_SWIZZLE_128B) &&
      sb::encode_tmap_2d(&td,
                         out_dt == SB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                           : (out_dt == SB_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32),
                         out, N, M, N * sb::dt_size(out_dt), 32, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) return cudaErrorInvalidValue;
  sbwide::WideParams p{};
  p.M = static_cast<int>(M);
  p.N = static_cast<int>(N);
  p.K = static_cast<int>(K);
  p.sa = sa;
  p.sb = sbp;
  p.post_scale = post;
  p.bias = (out_mode == sbtc::OUT_BF16 || out_mode == sbtc::OUT_F32) ? bias : nullptr;
  p.tiles_w = static_cast<int>(tiles_w);
  p.tiles_t = static_cast<int>(tiles_t);
#define SB_WIDE_CASE(KD, OM)                                                                    \
  if (kind == KD && out_mode == OM)                                                             \
    return sb_col ? launch_wide_t<KD, OM, true>(h, tw, tx, tx2, td, p, idesc)                   \
                  : launch_wide_t<KD, OM, false>(h, tw, tx, tx2, td, p, idesc);
  SB_WIDE_CASE(sbtc::KIND_I8, sbtc::OUT_BF16)
  SB_WIDE_CASE(sbtc::KIND_I8, sbtc::OUT_F32)
  SB_WIDE_CASE(sbtc::KIND_I8, sbtc::OUT_F32_EXACT)
  SB_WIDE_CASE(sbtc::KIND_I8, sbtc::OUT_I32)
  SB_WIDE_CASE(sbtc::KIND_F8, sbtc::OUT_BF16)
  SB_WIDE_CASE(sbtc::KIND_F8, sbtc::OUT_F32)
#undef SB_WIDE_CASE
  return cudaErrorNotSupported;
}

bool out_tmap(CUtensorMap* m, sb_dtype dt, void* out, int64_t M, int64_t N) {
  if (dt == SB_BF16)
    return sb::encode_tmap_2d(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, N, M, N * 2, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMapDataType t = dt == SB_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return sb::encode_tmap_2d(m, t, out, N, M, N * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
}

}  // namespace

namespace sb {

// The tensor-core GEMMs need TMA-legal operands (K % 16 == 0 for int8 / fp8, 16-byte aligned
// rows and bases). Anything else runs on the tiled SIMT kernels above, one to two orders of
// magnitude slower: say so once per process on stderr, and refuse outright when
// SB_STRICT_TC=1 (for callers that want a hard guarantee that the tcgen05 path ran).
sb_status simt_fallback(sb_handle h, const char* op, int64_t M, int64_t N, int64_t K) {
  static int strict = -1;
  if (strict < 0) strict = getenv("SB_STRICT_TC") ? atoi(getenv("SB_STRICT_TC")) : 0;
  if (strict)
    return fail(SB_ERR_UNSUPPORTED, op, "operands are not TMA-legal (K % 16, alignment); SB_STRICT_TC=1 forbids the SIMT path");
  static std::once_flag warned;
  std::call_once(warned, [&] {
    fprintf(stderr,
            "switchback_b200: %s %lldx%lldx%lld is not TMA-legal (needs K %% 16 == 0 and 16-byte aligned rows): "
            "running the SIMT fallback, much slower than tcgen05 (warned once; SB_STRICT_TC=1 makes it an error)\n",
            op, static_cast<long long>(M), static_cast<long long>(N), static_cast<long long>(K));
  });
  (void)h;
  return SB_OK;
}

bool encode_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  EncodeFn fn = get_encode();
  if (!fn) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

sb_status gemm_i8(sb_handle h, const int8_t* qa, const float* sa, const int8_t* qb, const float* sbp, int scale_mode,
                  int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt, int exact, const float* bias,
                  const void* resid, int64_t ld_resid) {
  const char* op = "int8 matmul";
  const bool raw = scale_mode == SB_SCALE_NONE;
  if (raw && out_dt != SB_I32 && out_dt != SB_I64) return fail(SB_ERR_INVALID_ARGUMENT, op, "raw output needs I32/I64");
  if (!raw && out_dt != SB_F32 && out_dt != SB_BF16) return fail(SB_ERR_INVALID_ARGUMENT, op, "bad output dtype");
  if (out_dt == SB_I32 && K > kInt32SafeInner)
    return fail(SB_ERR_INVALID_ARGUMENT, op, "int32 accumulator would overflow (k > 133144); use I64");
  const int sa_stride = 1;  // A is always row-wise (X or G)
  const int sb_stride = scale_mode == SB_SCALE_ROW_ROW ? 1 : 0;
  int out_mode;
  if (raw) out_mode = sbtc::OUT_I32;
  else if (out_dt == SB_BF16) out_mode = sbtc::OUT_BF16;
  else out_mode = exact ? sbtc::OUT_F32_EXACT : sbtc::OUT_F32;

  const bool tc_ok = out_dt != SB_I64 && K <= kInt32SafeInner && (K % 16 == 0) && aligned(qa, 16) &&
                     aligned(qb, 16) && aligned(out, 16) && ((N * static_cast<int64_t>(dt_size(out_dt))) % 16 == 0) &&
                     M < (1LL << 31) && N < (1LL << 31) && get_encode() != nullptr;
  CUtensorMap td;
  if (tc_ok && out_tmap(&td, out_dt, out, M, N)) {
    const Operand A{qa, CU_TENSOR_MAP_DATA_TYPE_UINT8, static_cast<uint64_t>(K), static_cast<uint64_t>(M),
                    static_cast<uint64_t>(K), false, 128};
    const Operand B{qb, CU_TENSOR_MAP_DATA_TYPE_UINT8, static_cast<uint64_t>(K), static_cast<uint64_t>(N),
                    static_cast<uint64_t>(K), false, 128};
    sbtc::Params p{};
    p.M = static_cast<int>(M);
    p.N = static_cast<int>(N);
    p.K = static_cast<int>(K);
    p.sa = sa;
    p.sb = sbp;
    p.sa_stride = sa_stride;
    p.sb_stride = sb_stride;
    p.post_scale = 1.0f / 16129.0f;
    p.splits = 1;
    p.bias = (out_mode == sbtc::OUT_BF16 || out_mode == sbtc::OUT_F32) ? bias : nullptr;
    if (resid == nullptr) {
      const cudaError_t we = launch_wide(h, sbtc::KIND_I8, out_mode, sb_stride == 1, qa, qb, M, N, K, sa, sbp,
                                         p.post_scale, bias, out, out_dt, 0);
      if (we == cudaSuccess) return SB_OK;
      if (we != cudaErrorNotSupported) return cuda_fail(op, we);
    }
    const bool fuse_resid = resid != nullptr && out_mode == sbtc::OUT_BF16 && aligned(resid, 4) && ld_resid % 2 == 0;
    p.resid = fuse_resid ? static_cast<const __nv_bfloat16*>(resid) : nullptr;
    p.ld_resid = ld_resid;
    cudaError_t e;
    const bool col = sb_stride == 1;
    switch (out_mode) {
      case sbtc::OUT_BF16:
        if (fuse_resid)
          e = col ? launch_tc<sbtc::KIND_I8, sbtc::OUT_BF16_RESID, false, false, true>(h, A, B, td, p, 0)
                  : launch_tc<sbtc::KIND_I8, sbtc::OUT_BF16_RESID>(h, A, B, td, p, 0);
        else
          e = col ? launch_tc<sbtc::KIND_I8, sbtc::OUT_BF16, false, false, true>(h, A, B, td, p, 0)
                  : launch_tc<sbtc::KIND_I8, sbtc::OUT_BF16>(h, A, B, td, p, 0);
        break;
      case sbtc::OUT_F32:
        e = col ? launch_tc<sbtc::KIND_I8, sbtc::OUT_F32, false, false, true>(h, A, B, td, p, 0)
                : launch_tc<sbtc::KIND_I8, sbtc::OUT_F32>(h, A, B, td, p, 0);
        break;
      case sbtc::OUT_F32_EXACT:
        e = col ? launch_tc<sbtc::KIND_I8, sbtc::OUT_F32_EXACT, false, false, true>(h, A, B, td, p, 0)
                : launch_tc<sbtc::KIND_I8, sbtc::OUT_F32_EXACT>(h, A, B, td, p, 0);
        break;
      default: e = launch_tc<sbtc::KIND_I8, sbtc::OUT_I32>(h, A, B, td, p, 0); break;
    }
    if (e != cudaSuccess) return cuda_fail(op, e);
    if (bias && !p.bias) {
      const cudaError_t be = launch_add_bias(h, out, out_dt, M, N, bias);
      if (be != cudaSuccess) return cuda_fail(op, be);
    }
    if (resid && !fuse_resid) {
      if (ld_resid != N) return fail(SB_ERR_UNSUPPORTED, op, "unfused residual must be contiguous");
      const cudaError_t re = launch_add_residual(h, out, out_dt, M, N, resid);
      if (re != cudaSuccess) return cuda_fail(op, re);
    }
    return SB_OK;
  }
  // SIMT path (unaligned / tiny / int64 accumulation)
  if (K <= kInt32SafeInner) {
    const sb_status fs = simt_fallback(h, op, M, N, K);
    if (fs != SB_OK) return fs;
  }
  const dim3 grid(static_cast<unsigned>((N + kSimtTile - 1) / kSimtTile),
                  static_cast<unsigned>(std::min<int64_t>((M + kSimtTile - 1) / kSimtTile, 65535)));
  h->launches++;
  if (out_dt == SB_I64)
    k_gemm_i8_simt<5><<<grid, 256, 0, h->stream>>>(qa, sa, sa_stride, qb, sbp, sb_stride, M, N, K, out);
  else if (out_mode == sbtc::OUT_I32)
    k_gemm_i8_simt<sbtc::OUT_I32><<<grid, 256, 0, h->stream>>>(qa, sa, sa_stride, qb, sbp, sb_stride, M, N, K, out);
  else if (out_mode == sbtc::OUT_F32_EXACT)
    k_gemm_i8_simt<sbtc::OUT_F32_EXACT><<<grid, 256, 0, h->stream>>>(qa, sa, sa_stride, qb, sbp, sb_stride, M, N, K,
                                                                     out);
  else if (out_mode == sbtc::OUT_F32)
    k_gemm_i8_simt<sbtc::OUT_F32><<<grid, 256, 0, h->stream>>>(qa, sa, sa_stride, qb, sbp, sb_stride, M, N, K, out);
  else
    k_gemm_i8_simt<sbtc::OUT_BF16><<<grid, 256, 0, h->stream>>>(qa, sa, sa_stride, qb, sbp, sb_stride, M, N, K, out);
  SB_LAUNCH_CHECK(op);
  if (bias) SB_CUDA_CHECK(op, launch_add_bias(h, out, out_dt, M, N, bias));
  if (resid) {
    if (ld_resid != N) return fail(SB_ERR_UNSUPPORTED, op, "unfused residual must be contiguous");
    SB_CUDA_CHECK(op, launch_add_residual(h, out, out_dt, M, N, resid));
  }
  return SB_OK;
}

sb_status matmul_f32_seq(sb_handle h, const float* a, int64_t a_rs, int64_t a_ks, const float* bt, int64_t b_rs,
                         int64_t b_ks, int64_t r, int64_t c, int64_t k, float* y, int accumulate) {
  const dim3 grid(static_cast<unsigned>((c + 63) / 64), static_cast<unsigned>((r + 63) / 64));
  h->launches++;
  k_matmul_seq<float><<<grid, 256, 0, h->stream>>>(a, a_rs, a_ks, bt, b_rs, b_ks, r, c, k, y, accumulate);
  SB_LAUNCH_CHECK("matmul");
  return SB_OK;
}

sb_status wgrad(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n, float* dw,
                int exact, int accumulate, const RowQuant* rq) {
  const char* op = "linear_backward";
  CUtensorMap td;
  // a fused row-wise quantize of G rides in the one-wave dW kernel (bf16 G, 16-byte rows);
  // anywhere else it is the standalone quantizer, launched first
  const bool fuse_q = rq && dt == SB_BF16 && !exact && !accumulate && m % 8 == 0 && aligned(g, 16) &&
                      aligned(rq->q, 16) && rq->ldq % 16 == 0;
  if (rq && !fuse_q) {
    const cudaError_t qe = launch_quantize_rowwise(h, g, dt, b, m, m, rq->q, rq->ldq, rq->state);
    if (qe != cudaSuccess) return cuda_fail(op, qe);
    rq = nullptr;
  }
  if (dt == SB_BF16 && !exact && (m % 8 == 0) && (n % 8 == 0) && aligned(g, 16) && aligned(x, 16) && aligned(dw, 16) &&
      b < (1LL << 31) && get_encode() != nullptr && out_tmap(&td, SB_F32, dw, m, n)) {
    // A = G[T x m] and B = X[T x n] read in place as MN-major operands; K = T tokens
    const Operand A{g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<uint64_t>(m), static_cast<uint64_t>(b),
                    static_cast<uint64_t>(m * 2), true, 64};
    const Operand B{x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<uint64_t>(n), static_cast<uint64_t>(b),
                    static_cast<uint64_t>(n * 2), true, 64};
    if (!accumulate) {
      const cudaError_t we = launch_dw_wide(h, A, B, td, m, n, b, rq);
      if (we == cudaSuccess) return SB_OK;
      if (we != cudaErrorNotSupported) return cuda_fail(op, we);
    }
    if (rq) {  // the one-wave kernel does not apply to this shape: quantize separately
      const cudaError_t qe = launch_quantize_rowwise(h, g, dt, b, m, m, rq->q, rq->ldq, rq->state);
      if (qe != cudaSuccess) return cuda_fail(op, qe);
      rq = nullptr;
    }
    sbtc::Params p{};
    p.M = static_cast<int>(m);
    p.N = static_cast<int>(n);
    p.K = static_cast<int>(b);
    p.post_scale = 1.0f;
    // Split K (= tokens) in two when the output has too few tiles to fill the SMs (pairs) in
    // whole waves: both halves reduce-add into a zeroed dW, and 0 + a + b == 0 + b + a, so the
    // result stays deterministic (more splits would make the fp32 sum order-dependent).
    const bool two = use_2cta(h, m, ((m + 255) / 256) * ((n + 255) / 256));
    const int tm = static_cast<int>((m + (two ? 256 : 128) - 1) / (two ? 256 : 128));
    const int tiles = tm * static_cast<int>((n + 255) / 256);
    const int slots = two ? h->num_sms / 2 : h->num_sms;
    const int64_t kblocks = (b + 63) / 64;
    auto eff = [&](int s) {
      const int u = tiles * s;
      const int w = (u + slots - 1) / slots;
      return double(u) / (double(w) * slots);
    };
    p.splits = (!accumulate && kblocks >= 64 && eff(2) > eff(1) + 0.05) ? 2 : 1;
    // raster so the larger operand is streamed once: tiles sharing a block of it run
    // concurrently (G^T X: walk M when X is the larger of the two)
    p.m_fast = n > m ? 1 : 0;
    cudaError_t e;
    if (p.splits == 2) {
      e = cudaMemsetAsync(dw, 0, sizeof(float) * m * n, h->stream);
      if (e == cudaSuccess) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW_ADD, true, true>(h, A, B, td, p, 0);
    } else {
      e = accumulate ? launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW_ADD, true, true>(h, A, B, td, p, 0)
                     : launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW, true, true>(h, A, B, td, p, 0);
    }
    if (e != cudaSuccess) return cuda_fail(op, e);
    return SB_OK;
  }
  // exact sequential (or unaligned fallback): dW[i][j] = sum_t G[t][i] * X[t][j]
  if (rq) {
    const cudaError_t qe = launch_quantize_rowwise(h, g, dt, b, m, m, rq->q, rq->ldq, rq->state);
    if (qe != cudaSuccess) return cuda_fail(op, qe);
  }
  if (!exact) {
    const sb_status fs = simt_fallback(h, op, m, n, b);
    if (fs != SB_OK) return fs;
  }
  const dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64));
  h->launches++;
  if (dt == SB_BF16)
    k_matmul_seq<__nv_bfloat16><<<grid, 256, 0, h->stream>>>(static_cast<const __nv_bfloat16*>(g), 1, m,
                                                             static_cast<const __nv_bfloat16*>(x), 1, n, m, n, b, dw,
                                                             accumulate);
  else
    k_matmul_seq<float><<<grid, 256, 0, h->stream>>>(static_cast<const float*>(g), 1, m, static_cast<const float*>(x), 1,
                                                     n, m, n, b, dw, accumulate);
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

bool dw_wide_serves(sb_handle h, int64_t m, int64_t n, int64_t b) {
  // the shape rule of launch_dw_wide (dw_wide_plan) with the device's co-resident pair count
  if (b <= 0 || b >= (1LL << 31) || m % 8 || n % 8) return false;
  const int max_pairs = dw_wide_pairs(h);
  if (max_pairs <= 0) return false;
  bool trans = false;
  return dw_wide_plan(max_pairs, m, n, &trans);
}

sb_status wgrad_reduce_scatter(sb_handle h, const void* g, const void* x, sb_dtype dt, int64_t b, int64_t m, int64_t n,
                               float* dw, const sb_symbuf& sym, const RowQuant* rq) {
  const char* op = "wgrad_reduce_scatter";
  if (sym.world < 1 || sym.world > 8 || !sym.opened) return fail(SB_ERR_INVALID_ARGUMENT, op, "symmetric buffer not opened");
  const bool ok = dt == SB_BF16 && m % 8 == 0 && n % 8 == 0 && aligned(g, 16) && aligned(x, 16) && aligned(dw, 16) &&
                  b > 0 && b < (1LL << 31) && get_encode() != nullptr &&
                  (!rq || (aligned(rq->q, 16) && rq->ldq % 16 == 0));
  if (!ok) return fail(SB_ERR_UNSUPPORTED, op, "bf16, m % 8 == 0, n % 8 == 0, 16-byte aligned operands");
  const size_t off = static_cast<size_t>(reinterpret_cast<const uint8_t*>(dw) - static_cast<const uint8_t*>(sym.local));
  sbdw::DMaps<8> dm{};
  dm.world = sym.world;
  dm.nblocks = static_cast<int>((m + 31) / 32);
  CUtensorMap td;
  if (!out_tmap(&td, SB_F32, dw, m, n)) return fail(SB_ERR_UNSUPPORTED, op, "tensor map encode failed");
  for (int r = 0; r < sym.world; ++r) {
    float* pr = reinterpret_cast<float*>(static_cast<uint8_t*>(sym.peer[r]) + off);
    if (!out_tmap(&dm.m[r], SB_F32, pr, m, n)) return fail(SB_ERR_UNSUPPORTED, op, "peer tensor map encode failed");
  }
  const Operand A{g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<uint64_t>(m), static_cast<uint64_t>(b),
                  static_cast<uint64_t>(m * 2), true, 64};
  const Operand B{x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, static_cast<uint64_t>(n), static_cast<uint64_t>(b),
                  static_cast<uint64_t>(n * 2), true, 64};
  const cudaError_t e = launch_dw_wide(h, A, B, td, m, n, b, rq, &dm);
  if (e == cudaErrorNotSupported)
    return fail(SB_ERR_UNSUPPORTED, op, "shape not served by the one-wave dW kernel (use sb_wgrad + all-reduce)");
  if (e != cudaSuccess) return cuda_fail(op, e);
  return SB_OK;
}

sb_status gemm_bf16_tc(sb_handle h, const void* a, bool a_mn, const void* b, bool b_mn, int64_t M, int64_t N, int64_t K,
                       void* out, sb_dtype out_dt, const float* one) {
  const char* op = "matmul";
  const bool tc_ok = (a_mn ? M % 8 == 0 : K % 8 == 0) && (b_mn ? N % 8 == 0 : K % 8 == 0) && aligned(a, 16) &&
                     aligned(b, 16) && aligned(out, 16) && ((N * static_cast<int64_t>(dt_size(out_dt))) % 16 == 0) &&
                     get_encode() != nullptr;
  CUtensorMap td;
  if (tc_ok && out_tmap(&td, out_dt, out, M, N)) {
    const CUtensorMapDataType bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const Operand A = a_mn ? Operand{a, bf, static_cast<uint64_t>(M), static_cast<uint64_t>(K), static_cast<uint64_t>(M * 2), true, 64}
                           : Operand{a, bf, static_cast<uint64_t>(K), static_cast<uint64_t>(M), static_cast<uint64_t>(K * 2), false, 64};
    const Operand B = b_mn ? Operand{b, bf, static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint64_t>(N * 2), true, 64}
                           : Operand{b, bf, static_cast<uint64_t>(K), static_cast<uint64_t>(N), static_cast<uint64_t>(K * 2), false, 64};
    sbtc::Params p{};
    p.M = static_cast<int>(M);
    p.N = static_cast<int>(N);
    p.K = static_cast<int>(K);
    p.sa = one;
    p.sb = one;
    p.post_scale = 1.0f;
    p.splits = 1;
    cudaError_t e;
    if (out_dt == SB_BF16) {
      if (!a_mn && !b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_BF16, false, false>(h, A, B, td, p, 0);
      else if (!a_mn && b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_BF16, false, true>(h, A, B, td, p, 0);
      else if (a_mn && !b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_BF16, true, false>(h, A, B, td, p, 0);
      else e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_BF16, true, true>(h, A, B, td, p, 0);
    } else {
      if (!a_mn && !b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW, false, false>(h, A, B, td, p, 0);
      else if (!a_mn && b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW, false, true>(h, A, B, td, p, 0);
      else if (a_mn && !b_mn) e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW, true, false>(h, A, B, td, p, 0);
      else e = launch_tc<sbtc::KIND_BF16, sbtc::OUT_F32_RAW, true, true>(h, A, B, td, p, 0);
    }
    if (e != cudaSuccess) return cuda_fail(op, e);
    return SB_OK;
  }
  // any shape: fp32-accumulating SIMT kernel over the same index maps
  {
    const sb_status fs = simt_fallback(h, op, M, N, K);
    if (fs != SB_OK) return fs;
  }
  const __nv_bfloat16* Ap = static_cast<const __nv_bfloat16*>(a);
  const __nv_bfloat16* Bp = static_cast<const __nv_bfloat16*>(b);
  const int64_t a_rs = a_mn ? 1 : K, a_ks = a_mn ? M : 1, b_rs = b_mn ? 1 : K, b_ks = b_mn ? N : 1;
  const dim3 grid(static_cast<unsigned>((N + 63) / 64), static_cast<unsigned>((M + 63) / 64));
  h->launches++;
  if (out_dt == SB_BF16)
    k_matmul_seq<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, h->stream>>>(Ap, a_rs, a_ks, Bp, b_rs, b_ks, M, N, K,
                                                                            static_cast<__nv_bfloat16*>(out), 0);
  else
    k_matmul_seq<__nv_bfloat16, float><<<grid, 256, 0, h->stream>>>(Ap, a_rs, a_ks, Bp, b_rs, b_ks, M, N, K,
                                                                    static_cast<float*>(out), 0);
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

sb_status gemm_fp8(sb_handle h, const uint8_t* qa, int fa, const float* sa, int axa, const uint8_t* qb, int fb,
                   const float* sbp, int axb, int64_t M, int64_t N, int64_t K, void* out, sb_dtype out_dt) {
  const char* op = "fp8 matmul";
  if (out_dt != SB_F32 && out_dt != SB_BF16) return fail(SB_ERR_INVALID_ARGUMENT, op, "bad output dtype");
  const int sa_stride = axa == SB_AXIS_ROW ? 1 : 0, sb_stride = axb == SB_AXIS_ROW ? 1 : 0;
  const bool tc_ok = (K % 16 == 0) && aligned(qa, 16) && aligned(qb, 16) && aligned(out, 16) &&
                     ((N * static_cast<int64_t>(dt_size(out_dt))) % 16 == 0) && get_encode() != nullptr;
  CUtensorMap td;
  if (tc_ok && out_tmap(&td, out_dt, out, M, N)) {
    const Operand A{qa, CU_TENSOR_MAP_DATA_TYPE_UINT8, static_cast<uint64_t>(K), static_cast<uint64_t>(M),
                    static_cast<uint64_t>(K), false, 128};
    const Operand B{qb, CU_TENSOR_MAP_DATA_TYPE_UINT8, static_cast<uint64_t>(K), static_cast<uint64_t>(N),
                    static_cast<uint64_t>(K), false, 128};
    sbtc::Params p{};
    p.M = static_cast<int>(M);
    p.N = static_cast<int>(N);
    p.K = static_cast<int>(K);
    p.sa = sa;
    p.sb = sbp;
    p.sa_stride = sa_stride;
    p.sb_stride = sb_stride;
    p.post_scale = 1.0f;
    p.splits = 1;
    const uint32_t idesc = sbtc::KindTraits<sbtc::KIND_F8>::IDESC | (static_cast<uint32_t>(fa) << 7) |
                           (static_cast<uint32_t>(fb) << 10);
    if (sa_stride == 1) {  // transposed wide kernel: W (format fb) is the MMA's A operand, X (fa) its B
      const uint32_t idesc_t = sbtc::KindTraits<sbtc::KIND_F8>::IDESC | (static_cast<uint32_t>(fb) << 7) |
                               (static_cast<uint32_t>(fa) << 10);
      const cudaError_t we = launch_wide(h, sbtc::KIND_F8, out_dt == SB_BF16 ? sbtc::OUT_BF16 : sbtc::OUT_F32,
                                         sb_stride == 1, qa, qb, M, N, K, sa, sbp, 1.0f, nullptr, out, out_dt, idesc_t);
      if (we == cudaSuccess) return SB_OK;
      if (we != cudaErrorNotSupported) return cuda_fail(op, we);
    }
    cudaError_t e;
    if (sb_stride)
      e = out_dt == SB_BF16 ? launch_tc<sbtc::KIND_F8, sbtc::OUT_BF16, false, false, true>(h, A, B, td, p, idesc)
                            : launch_tc<sbtc::KIND_F8, sbtc::OUT_F32, false, false, true>(h, A, B, td, p, idesc);
    else
      e = out_dt == SB_BF16 ? launch_tc<sbtc::KIND_F8, sbtc::OUT_BF16>(h, A, B, td, p, idesc)
                            : launch_tc<sbtc::KIND_F8, sbtc::OUT_F32>(h, A, B, td, p, idesc);
    if (e != cudaSuccess) return cuda_fail(op, e);
    return SB_OK;
  }
  {
    const sb_status fs = simt_fallback(h, op, M, N, K);
    if (fs != SB_OK) return fs;
  }
  const dim3 grid(static_cast<unsigned>((N + 127) / 128), static_cast<unsigned>(std::min<int64_t>(M, 65535)));
  h->launches++;
  k_gemm_fp8_simt<<<grid, 128, 0, h->stream>>>(qa, fa, sa, sa_stride, qb, fb, sbp, sb_stride, M, N, K, out,
                                               out_dt == SB_BF16);
  SB_LAUNCH_CHECK(op);
  return SB_OK;
}

}  // namespace sb
