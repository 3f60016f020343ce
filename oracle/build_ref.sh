#!/usr/bin/env bash
# Build the CPU oracles.  TEST INFRASTRUCTURE ONLY.
#
#   oracle/_build/liborc.so  the C restatement (oracle/hcc_oracle.c); always built.
#   oracle/_ref/libhcc_ref.so  the UNMODIFIED reference library, compiled
#       directly from its own sources where they lie under /root/reference
#       (nothing is copied into this repo), plus oracle/ref_capi.cpp.  Built
#       only when /root/reference exists (the dev container); the GPU box
#       receives the prebuilt .so with the gpurun snapshot.
#
# Flags follow the reference build: C++20, OpenMP, -ffp-contract=off
# (proj/CMakeLists.txt:15-17, proj/src/CMakeLists.txt:13).  The reference
# CMake itself is not used: it requires GTest (proj/CMakeLists.txt:13), which
# is absent here.
set -euo pipefail
here="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
mkdir -p "$here/_build"
gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared -Wall \
    -o "$here/_build/liborc.so.tmp" "$here/hcc_oracle.c" -lm
mv "$here/_build/liborc.so.tmp" "$here/_build/liborc.so"

REF="${HCC_REFERENCE:-/root/reference}/proj"
if [ -d "$REF/src" ]; then
  mkdir -p "$here/_ref"
  g++ -std=c++20 -O2 -fopenmp -ffp-contract=off -fPIC -shared \
      -I "$REF/include" -I "$REF/src" -I "$REF/tests" \
      "$REF/src/codec.cpp" "$REF/src/codec_omp.cpp" "$REF/src/codec_serial.cpp" \
      "$REF/src/collectives.cpp" "$REF/src/netsim.cpp" "$REF/src/parallel3d.cpp" \
      "$REF/src/toymodel.cpp" "$REF/src/linalg.cpp" \
      "$REF/tests/support/oracles.cpp" "$here/ref_capi.cpp" \
      -o "$here/_ref/libhcc_ref.so.tmp"
  mv "$here/_ref/libhcc_ref.so.tmp" "$here/_ref/libhcc_ref.so"
fi
