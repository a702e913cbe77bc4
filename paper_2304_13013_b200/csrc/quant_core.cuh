// quant_core.cuh — the exact row-wise int8 quantizer's element and row primitives, shared by
// the standalone quantize kernels (quantize.cu, K1) and the kernels that fuse a row-wise
// quantize into another launch (the dW GEMM, tc_dw_wide.cuh). See quantize.cu's header for
// why the payload is bit-exact against quantize.cpp:116-133.
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace sbq {

constexpr uint32_t kNonFiniteBits = 0x7f800000u;

__device__ __forceinline__ void raise_nonfinite(uint32_t* err) { atomicOr(err, 1u); }

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

template <typename T>
__device__ __forceinline__ uint32_t abs_bits(T v);
template <>
__device__ __forceinline__ uint32_t abs_bits<float>(float v) {
  return __float_as_uint(v) & 0x7fffffffu;
}
template <>
__device__ __forceinline__ uint32_t abs_bits<__nv_bfloat16>(__nv_bfloat16 v) {
  return (static_cast<uint32_t>(__bfloat16_as_ushort(v)) & 0x7fffu) << 16;
}

// Max of |x| bit patterns in a 16-byte vector, in fp32 bit space.
template <typename T>
__device__ __forceinline__ uint32_t vec_absmax_bits(const uint4& v);
template <>
__device__ __forceinline__ uint32_t vec_absmax_bits<float>(const uint4& v) {
  uint32_t a = max(v.x & 0x7fffffffu, v.y & 0x7fffffffu);
  uint32_t b = max(v.z & 0x7fffffffu, v.w & 0x7fffffffu);
  return max(a, b);
}
template <>
__device__ __forceinline__ uint32_t vec_absmax_bits<__nv_bfloat16>(const uint4& v) {
  uint32_t m = __vmaxu2(__vmaxu2(v.x & 0x7fff7fffu, v.y & 0x7fff7fffu), __vmaxu2(v.z & 0x7fff7fffu, v.w & 0x7fff7fffu));
  return max(m & 0xffffu, m >> 16) << 16;
}

struct Scale {
  float s;     // state after exact power-of-two prescale
  float inv;   // 127 / s (fp32, approximate is fine: only seeds the candidate)
  float pre;   // the power-of-two prescale applied to |x| and s
  float inv2;  // 127 / s * (1 + [2^-23, 2^-20]): the bf16 one-FMA exact path (see qvec)
};

__device__ __forceinline__ Scale make_scale(float state) {
  Scale sc;
  sc.pre = 1.0f;
  if (state < 0x1p-60f) sc.pre = 0x1p64f;
  else if (state > 0x1p64f) sc.pre = 0x1p-64f;
  sc.s = __fmul_rn(state, sc.pre);
  sc.inv = __fdiv_rn(127.0f, sc.s);
  sc.inv2 = __fmul_ru(__fdiv_ru(127.0f, sc.s), 1.0f + 0x1p-22f);
  return sc;
}

// |payload| = round_half_away(127|x|/s), exact (see file header).
template <bool kExactF32Products>
__device__ __forceinline__ float q_magnitude(float ax, const Scale& sc) {
  const float a = __fmul_rn(ax, sc.pre);
  const float qa = __fmul_rn(a, sc.inv);
  float k = floorf(__fadd_rn(qa, 0.5f));
  if (kExactF32Products) {
    const float num = __fmul_rn(127.0f, a);
    const float hi = __fmul_rn(__fadd_rn(k, 0.5f), sc.s);
    const float lo = __fmul_rn(__fsub_rn(k, 0.5f), sc.s);
    k = num >= hi ? __fadd_rn(k, 1.0f) : (num < lo ? __fsub_rn(k, 1.0f) : k);
  } else {
    const float frac = __fsub_rn(qa, floorf(qa));
    if (fabsf(__fsub_rn(frac, 0.5f)) < 1e-3f) {
      const double num = __dmul_rn(127.0, (double)a);
      const double hi = __dmul_rn((double)k + 0.5, (double)sc.s);
      const double lo = __dmul_rn((double)k - 0.5, (double)sc.s);
      k = num >= hi ? k + 1.0f : (num < lo ? k - 1.0f : k);
    }
  }
  return fminf(k, 127.0f);
}

template <typename T>
__device__ __forceinline__ int8_t quantize_one(T v, const Scale& sc) {
  const float x = to_f32(v);
  const float k = q_magnitude<sizeof(T) == 2>(fabsf(x), sc);
  const int ki = static_cast<int>(k);
  return static_cast<int8_t>(x < 0.0f ? -ki : ki);
}

__device__ __forceinline__ float state_from_bits(uint32_t bits) {
  return bits == 0u ? 1.0f : __uint_as_float(bits);  // all-zero slice sentinel (quantize.cpp:109-111)
}

// Pack the payload of one 16-byte input vector.
template <typename T>
struct VecQ;
template <>
struct VecQ<__nv_bfloat16> {
  using Out = uint2;  // 8 int8
  static __device__ __forceinline__ Out run(const uint4& v, const Scale& sc) {
    const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) lo |= (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(e[i], sc)))) << (8 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      hi |= (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(e[4 + i], sc)))) << (8 * i);
    return make_uint2(lo, hi);
  }
};
template <>
struct VecQ<float> {
  using Out = uint32_t;  // 4 int8
  static __device__ __forceinline__ Out run(const uint4& v, const Scale& sc) {
    const float* e = reinterpret_cast<const float*>(&v);
    uint32_t w = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) w |= (static_cast<uint32_t>(static_cast<uint8_t>(quantize_one(e[i], sc)))) << (8 * i);
    return w;
  }
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ------------------------------------------------------- vector payload ----
// Per element (fast path): qs = x * (127/s) (signed, fp32), m = qs + 1.5*2^23 rounds qs to
// the nearest integer and leaves it (two's complement) in the low byte of m; the residual
// r = qs - (m - 1.5*2^23) is exact. The candidate can only differ from the reference's
// round-half-away of the exact 127x/s when |r| is within ~2^-16 of 1/2, so a warp with any
// |r| > 1/2 - 2^-15 in the vector re-derives the vector with the exact comparison
// (q_magnitude). Bytes are packed with PRMT.
template <typename T>
struct Unpack;
template <>
struct Unpack<__nv_bfloat16> {
  static constexpr int N = 8;
  static __device__ __forceinline__ void run(const uint4& v, float (&x)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[2 * i] = __uint_as_float(w[i] << 16);
      x[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
};
template <>
struct Unpack<float> {
  static constexpr int N = 4;
  static __device__ __forceinline__ void run(const uint4& v, float (&x)[4]) {
    x[0] = __uint_as_float(v.x);
    x[1] = __uint_as_float(v.y);
    x[2] = __uint_as_float(v.z);
    x[3] = __uint_as_float(v.w);
  }
};

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23

__device__ __forceinline__ uint32_t pack4u(uint32_t u0, uint32_t u1, uint32_t u2, uint32_t u3) {
  return __byte_perm(__byte_perm(u0, u1, 0x0040), __byte_perm(u2, u3, 0x0040), 0x5410);
}

// bf16 input, one FMA per element, exact without any tie check. x and s are bf16 values
// (8 significant bits, s = max|x| >= |x|), so when 127|x|/s is not a half-integer it is at
// least (127|x|/s) * 2^-16 away from one: with x = a 2^e (a < 256 integer) and s = b 2^f
// (f >= e), 127|x|/s - (k + 1/2) = 2^e (254 a - (2k+1) b 2^(f-e)) / (2s), a nonzero multiple
// of 2^e / (2s) = (127|x|/s) / (254 a). inv2 = 127/s (1 + d) with 2^-23 < d < 2^-20, so
// x * inv2 (one rounding, fused with the magic add) moves the quotient by less than 2^-19 of
// itself — never across a half-integer — and moves exact ties strictly AWAY from zero, where
// round-to-nearest-even then lands on the reference's lround (round half away from zero).
__device__ __forceinline__ uint2 qvec_bf16_fast(const uint4& v, float inv2) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t u[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    u[2 * i] = __float_as_uint(__fmaf_rn(__uint_as_float(w[i] << 16), inv2, kMagic));
    u[2 * i + 1] = __float_as_uint(__fmaf_rn(__uint_as_float(w[i] & 0xffff0000u), inv2, kMagic));
  }
  return make_uint2(pack4u(u[0], u[1], u[2], u[3]), pack4u(u[4], u[5], u[6], u[7]));
}

// Quantize one 16-byte vector; `plain` = the row needs no power-of-two prescale.
template <typename T>
__device__ __forceinline__ typename VecQ<T>::Out qvec(const uint4& v, const Scale& sc, bool plain) {
  if constexpr (sizeof(T) == 2) {
    if (__all_sync(0xffffffffu, plain)) return qvec_bf16_fast(v, sc.inv2);
  }
  constexpr int N = Unpack<T>::N;
  float x[N];
  uint32_t u[N];
  Unpack<T>::run(v, x);
  float rmax = 0.0f;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const float qs = __fmul_rn(x[i], sc.inv);
    const float m = __fadd_rn(qs, kMagic);
    const float r = __fsub_rn(qs, __fsub_rn(m, kMagic));
    rmax = fmaxf(rmax, fabsf(r));
    u[i] = __float_as_uint(m);
  }
  // |qs - 127x/s| <= 127 * 2^-23 < 2^-16: only residuals within 2^-15 of 1/2 can round differently
  const bool near = !plain || rmax > 0.499969482421875f;  // 1/2 - 2^-15
  if (__any_sync(0xffffffffu, near)) {
#pragma unroll
    for (int i = 0; i < N; ++i)
      u[i] = __float_as_uint(__fadd_rn(copysignf(q_magnitude<sizeof(T) == 2>(fabsf(x[i]), sc), x[i]), kMagic));
  }
  if constexpr (N == 8) {
    return make_uint2(pack4u(u[0], u[1], u[2], u[3]), pack4u(u[4], u[5], u[6], u[7]));
  } else {
    return pack4u(u[0], u[1], u[2], u[3]);
  }
}

// One warp quantizes one row held in registers: VPL 16-byte vectors per lane, all loads issued
// before the first use, warp-reduced absmax, payload from the same registers (K1's row body,
// quantize.cpp:116-133). Non-finite rows latch `err` and store the offending bit pattern as the
// state (the reference throws, quantize.cpp:17-20).
template <typename T, int VPL>
__device__ __forceinline__ void quantize_row_reg(const uint4* __restrict__ xr, int nvec, int8_t* __restrict__ qrow,
                                                 float* __restrict__ state_row, uint32_t* err, int lane) {
  using Out = typename VecQ<T>::Out;
  uint4 v[VPL];
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int i = j * 32 + lane;
    v[j] = i < nvec ? ld_stream(xr + i) : make_uint4(0, 0, 0, 0);
  }
  uint32_t amax = 0;
#pragma unroll
  for (int j = 0; j < VPL; ++j) amax = max(amax, vec_absmax_bits<T>(v[j]));
  amax = __reduce_max_sync(0xffffffffu, amax);
  if (amax >= kNonFiniteBits) {
    if (lane == 0) {
      raise_nonfinite(err);
      *state_row = __uint_as_float(amax);
    }
    return;
  }
  const float st = state_from_bits(amax);
  if (lane == 0) *state_row = st;
  const Scale sc = make_scale(st);
  const bool plain = sc.pre == 1.0f;
  Out* qr = reinterpret_cast<Out*>(qrow);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    if (j * 32 >= nvec) break;  // warp-uniform (qvec votes across the warp)
    const int i = j * 32 + lane;
    const Out o = qvec<T>(v[j], sc, plain);
    if (i < nvec) qr[i] = o;
  }
}

// Any row length (16-byte vectorisable): absmax pass, then the payload pass re-reads the row
// (an L2 hit).
template <typename T>
__device__ __forceinline__ void quantize_row_stream(const uint4* __restrict__ xr, int64_t nvec, int8_t* __restrict__ qrow,
                                                    float* __restrict__ state_row, uint32_t* err, int lane) {
  using Out = typename VecQ<T>::Out;
  uint32_t amax = 0;
  for (int64_t v = lane; v < nvec; v += 32) amax = max(amax, vec_absmax_bits<T>(__ldg(xr + v)));
  amax = __reduce_max_sync(0xffffffffu, amax);
  if (amax >= kNonFiniteBits) {
    if (lane == 0) {
      raise_nonfinite(err);
      *state_row = __uint_as_float(amax);
    }
    return;
  }
  const float s = state_from_bits(amax);
  if (lane == 0) *state_row = s;
  const Scale sc = make_scale(s);
  const bool plain = sc.pre == 1.0f;
  Out* qr = reinterpret_cast<Out*>(qrow);
  for (int64_t b = 0; b < nvec; b += 32) {  // warp-uniform trip count (qvec votes)
    const int64_t v = b + lane;
    const Out o = qvec<T>(v < nvec ? __ldg(xr + v) : make_uint4(0, 0, 0, 0), sc, plain);
    if (v < nvec) qr[v] = o;
  }
}

// Compact bf16 row quantizer for kernels that carry it as a side task (the dW GEMM): the same
// payload / states as quantize_row_reg, but two passes over the row (absmax, then payload; the
// second read is an L2 hit) with U vectors per lane in flight per step, and the exact fallback
// out of line, so the side task adds a few hundred instructions to the host kernel instead of
// a fully unrolled row (a 64 KB kernel thrashed the instruction cache of the GEMM's issuing
// threads: ncu showed instruction-fetch requests at 65% of peak and the tensor pipe losing 12%).
static __device__ __noinline__ uint2 qvec_bf16_slow(uint4 v, Scale sc, bool plain) {
  return qvec<__nv_bfloat16>(v, sc, plain);
}
template <int U>
__device__ __forceinline__ void quantize_row_bf16_2pass(const uint4* __restrict__ xr, int nvec, int8_t* __restrict__ qrow,
                                                        float* __restrict__ state_row, uint32_t* err, int lane) {
  uint32_t amax = 0;
#pragma unroll 1
  for (int b = 0; b < nvec; b += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = b + j * 32 + lane;
      v[j] = i < nvec ? ld_stream(xr + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) amax = max(amax, vec_absmax_bits<__nv_bfloat16>(v[j]));
  }
  amax = __reduce_max_sync(0xffffffffu, amax);
  if (amax >= kNonFiniteBits) {
    if (lane == 0) {
      raise_nonfinite(err);
      *state_row = __uint_as_float(amax);
    }
    return;
  }
  const float st = state_from_bits(amax);
  if (lane == 0) *state_row = st;
  const Scale sc = make_scale(st);
  const bool plain = sc.pre == 1.0f;
  const bool fast = __all_sync(0xffffffffu, plain);
  uint2* qr = reinterpret_cast<uint2*>(qrow);
#pragma unroll 1
  for (int b = 0; b < nvec; b += 32 * U) {
    uint4 v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = b + j * 32 + lane;
      v[j] = i < nvec ? ld_stream(xr + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int i = b + j * 32 + lane;
      if (b + j * 32 >= nvec) break;  // warp-uniform
      const uint2 o = fast ? qvec_bf16_fast(v[j], sc.inv2) : qvec_bf16_slow(v[j], sc, plain);
      if (i < nvec) qr[i] = o;
    }
  }
}

}  // namespace sbq
