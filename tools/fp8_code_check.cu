// fp8_code_check.cu — exhaustive check of the packed fp8 magnitude coder of the bf16 fast path
// (quantize.cu fp8_code2_abs: FFMA2 / FADD2.RU ceil(n - 1/2) for the subnormal range, the folded
// integer add for normals) against the reference rounding (quantize.cpp:65-76: the mantissa
// rounded half toward zero), for EVERY fp32 magnitude in [0, 1] (the fast path's quotient range),
// e4m3 and e5m2. Prints the mismatch counts; both must be 0.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false tools/fp8_code_check.cu -o build/fp8_code_check
#include <cstdio>

// reference: floor-based snap of fp8_div_check.cu (no saturation: |a| <= 1)
template <int MB, int BIAS>
__device__ __forceinline__ unsigned ref_code(float a) {
  if (a < __uint_as_float(static_cast<unsigned>(128 - BIAS) << 23)) {
    const float n = __fmul_rn(a, __uint_as_float(static_cast<unsigned>(127 + BIAS + MB - 1) << 23));
    const float fl = floorf(n);
    return static_cast<unsigned>(fl) + (__fsub_rn(n, fl) > 0.5f ? 1u : 0u);
  }
  constexpr unsigned drop = 23 - MB;
  const unsigned rnd = (__float_as_uint(a) + (1u << (drop - 1)) - 1u) >> drop;
  return (((rnd >> MB) - 127u + BIAS) << MB) | (rnd & ((1u << MB) - 1u));
}

// the production coder (copy of quantize.cu fp8_code2_abs)
template <int MB, int BIAS>
__device__ __forceinline__ void code2(float2 a, unsigned& c0, unsigned& c1) {
  constexpr unsigned drop = 23 - MB;
  constexpr unsigned K = (1u << (drop - 1)) - 1u - (static_cast<unsigned>(127 - BIAS) << 23);
  constexpr unsigned thr = static_cast<unsigned>(128 - BIAS) << 23;
  const float P = __uint_as_float(static_cast<unsigned>(127 + BIAS + MB - 1) << 23);
  const float2 t = __ffma2_rn(a, make_float2(P, P), make_float2(-0.5f, -0.5f));
  const float2 m = __fadd2_ru(t, make_float2(12582912.0f, 12582912.0f));
  const unsigned ab0 = __float_as_uint(a.x), ab1 = __float_as_uint(a.y);
  c0 = ab0 < thr ? __float_as_uint(m.x) - 0x4B400000u : (ab0 + K) >> drop;
  c1 = ab1 < thr ? __float_as_uint(m.y) - 0x4B400000u : (ab1 + K) >> drop;
}

__global__ void k(unsigned long long* bad) {
  unsigned long long b4 = 0, b5 = 0;
  const unsigned n = 0x3F800000u + 1u;  // every magnitude 0 .. 1.0
  for (unsigned i = 2 * (blockIdx.x * blockDim.x + threadIdx.x); i < n; i += 2 * gridDim.x * blockDim.x) {
    const float2 a = make_float2(__uint_as_float(i), __uint_as_float(i + 1 < n ? i + 1 : i));
    unsigned c0, c1;
    code2<3, 7>(a, c0, c1);
    b4 += (c0 != ref_code<3, 7>(a.x)) + (c1 != ref_code<3, 7>(a.y));
    code2<2, 15>(a, c0, c1);
    b5 += (c0 != ref_code<2, 15>(a.x)) + (c1 != ref_code<2, 15>(a.y));
  }
  atomicAdd(&bad[0], b4);
  atomicAdd(&bad[1], b5);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  k<<<148 * 8, 256>>>(d);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("fp8 coder mismatches over all fp32 magnitudes in [0, 1]: e4m3 %llu, e5m2 %llu\n", h[0], h[1]);
  return (h[0] || h[1]) ? 1 : 0;
}
