#!/usr/bin/env bash
# Compile the reference's OWN unit-test sources (read in place from /root/reference/proj/tests,
# never copied) against the B200 lowprec shim (liblowprec_b200.so) + the minimal gtest header.
# Outputs go to build/reftests/ (git-ignored; the binaries travel to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF=${REF:-/root/reference/proj/tests}
OUT="$ROOT/build/reftests"
PKG="$ROOT/paper_2304_13013_b200"
if [ ! -d "$REF" ]; then echo "reference tests absent; keeping prebuilt $OUT"; exit 0; fi
mkdir -p "$OUT"
for t in matrix_test quantize_test linear_test optimizer_test; do
  g++ -O1 -std=c++20 -ffp-contract=off -I "$HERE" -I "$PKG/csrc/shim_include" -I "$PKG/csrc" -I "$ROOT/include" \
      "$REF/$t.cpp" "$HERE/main.cpp" -o "$OUT/$t" -L "$PKG" -llowprec_b200 -lswitchback_b200 \
      -Wl,-rpath,"$PKG" -Wl,-rpath,'$ORIGIN/../../paper_2304_13013_b200'
done
echo "built reference unit tests into $OUT"
