#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Compiles the UNMODIFIED reference transform path
# (proj/src/{transform,soe,rng}.cpp) where it lies under /root/reference, with
# the same flags as proj/CMakeLists.txt:29-33 (-std=c++20 -O2), together with
# oracle/ref_capi.cpp (extern "C" shim + table-backed cf_soe).  Output goes only
# to oracle/_ref/ (git-ignored, but NOT gpurun-ignored, so it travels to the GPU
# box).  cf.cpp / reduction.cpp need Eigen (absent) and are not built.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${FGT1D_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -f "$REF/src/transform.cpp" ]; then
  echo "reference sources not found at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT"
g++ -std=c++20 -O2 -fPIC -shared -pthread -fext-numeric-literals \
  -I"$REF/include" -I"$REF/src" \
  "$REF/src/transform.cpp" "$REF/src/soe.cpp" "$REF/src/rng.cpp" \
  "$HERE/ref_capi.cpp" -o "$OUT/libfgt1d_ref.so.tmp"
mv "$OUT/libfgt1d_ref.so.tmp" "$OUT/libfgt1d_ref.so"
echo "built $OUT/libfgt1d_ref.so"
