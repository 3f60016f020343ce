#!/usr/bin/env bash
# Builds the reference's OWN test suite and trainer against the B200 drop-in:
#   /root/reference/proj/tests/*.cpp + tests/support/*.cpp      (unchanged)
#   /root/reference/proj/src/{toymodel,linalg}.cpp              (unchanged;
#       the trainer and its fp32 math are outside the hot path)
# compiled with include/hcc/ (this repo) FIRST on the include path, so every
# hot-path header (codec, collectives, netsim, parallel3d, comm_path, errors,
# rng) is the drop-in's, and linked against libhcc_b200.so -> libhccx.so
# instead of the reference library.  GoogleTest is not in the image: the
# stand-in tests/cpp/gtest/gtest.h provides the macros the suite uses.
# Output: tests/cpp/_refbuild/hcc_ref_tests (git-ignored; travels to the GPU
# box with gpurun, where tests/test_refsuite_gpu.py runs it).  Nothing here
# runs without /root/reference (the GPU box only uses the prebuilt binary).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../../.." && pwd)"
REF="${HCC_REFERENCE:-/root/reference}/proj"
OUT="$ROOT/tests/cpp/_refbuild"
if [ ! -d "$REF/tests" ]; then
  echo "refsuite: $REF absent, keeping the prebuilt $OUT/hcc_ref_tests"
  exit 0
fi
CXX=g++  # the system g++ (libgomp for the reference library; $CXX may point elsewhere)

# compile <objdir> <stamp-header> <flags...> -- <sources...>
compile() {
  local dir="$1" stamp="$2"
  shift 2
  local flags=()
  while [ "$1" != "--" ]; do flags+=("$1"); shift; done
  shift
  mkdir -p "$dir"
  OBJS=()
  for s in "$@"; do
    local o="$dir/$(basename "${s%.cpp}").o"
    OBJS+=("$o")
    if [ ! -f "$o" ] || [ "$s" -nt "$o" ] || [ "$stamp" -nt "$o" ]; then
      "$CXX" -std=c++20 -O2 -ffp-contract=off -w "${flags[@]}" -c "$s" -o "$o" &
    fi
  done
  wait
}

SUITE=("$REF"/tests/test_*.cpp "$REF"/tests/support/*.cpp "$ROOT/tests/cpp/gtest/gtest_main.cpp")

# (1) the suite + the reference trainer against the B200 drop-in
compile "$OUT" "$ROOT/include/hcc/hcc_b200.hpp" -I"$ROOT/include" -I"$ROOT/tests/cpp" -I"$REF/include" -I"$REF/tests" \
  -- "${SUITE[@]}" "$REF/src/toymodel.cpp" "$REF/src/linalg.cpp"
"$CXX" -o "$OUT/hcc_ref_tests" "${OBJS[@]}" -L"$ROOT/paper_2409_02423_b200" -lhcc_b200 -lhccx \
  -Wl,-rpath,'$ORIGIN/../../../paper_2409_02423_b200'
echo "refsuite: built $OUT/hcc_ref_tests"

# (2) the same suite against the reference's own library (every src/*.cpp,
# OpenMP, CPU): its pass/fail record is what the drop-in must reproduce
compile "$OUT/reflib" "$REF/include/hcc/codec.hpp" -fopenmp -I"$REF/include" -I"$ROOT/tests/cpp" -I"$REF/tests" -I"$REF/src" \
  -- "${SUITE[@]}" "$REF"/src/*.cpp
"$CXX" -fopenmp -o "$OUT/hcc_ref_tests_reflib" "${OBJS[@]}"
echo "refsuite: built $OUT/hcc_ref_tests_reflib"
