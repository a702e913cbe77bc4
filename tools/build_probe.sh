#!/usr/bin/env bash
# Build the pipeline-probe binary (all csrc + tools/gemm_probe.cu, -DSB_GEMM_PROBE) into build/.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
C="$ROOT/paper_2304_13013_b200/csrc"
mkdir -p "$ROOT/build/probe"
cat > "$ROOT/build/probe/probe_glue.cu" <<'EOG'
#include <cuda_runtime.h>
#include "tc_gemm.cuh"
namespace sbtc { __device__ unsigned long long g_probe[1024 * 6]; __device__ long long g_trace[4096]; __device__ unsigned long long g_probe_ns[1024]; }
extern "C" void sb_probe_ns_read(unsigned long long* out, int n) { cudaMemcpyFromSymbol(out, sbtc::g_probe_ns, n * 8); }
extern "C" void sb_trace_read(long long* out) { cudaMemcpyFromSymbol(out, sbtc::g_trace, 4096 * 8); }
extern "C" void sb_probe_read(unsigned long long* out, int n) { cudaMemcpyFromSymbol(out, sbtc::g_probe, n * 8); }
extern "C" void sb_probe_reset() { static unsigned long long z[1024 * 6] = {0}; cudaMemcpyToSymbol(sbtc::g_probe, z, sizeof(z)); }
EOG
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -rdc=true --fmad=false -DSB_GEMM_PROBE $EXTRA -I "$ROOT/include" -I "$C" \
  "$C/quantize.cu" "$C/gemm.cu" "$C/optim.cu" "$C/capi.cu" "$C/util.cu" "$C/dp.cu" "$ROOT/build/probe/probe_glue.cu" \
  "$ROOT/tools/gemm_probe.cu" -o "$ROOT/build/gemm_probe$SUFFIX" -ldl -lcuda
echo built build/gemm_probe
