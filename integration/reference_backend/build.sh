#!/bin/bash
# Build the reference's own acceptance gate and unit tests with the B200
# path registered as the first backend of the reference roster (INTEGRATION.md
# §3), from the reference checkout (read-only, REF) and this repository.
# Outputs go only to baseline/accept/ (git-ignored; it travels to the GPU
# box with the snapshot):
#   acceptance   proj/tests/acceptance.cpp -- the 8-criterion release gate
#   unit_tests   proj/tests/test_{lookup,oracle,tables}.cpp, unchanged, with
#                the doctest stand-in of doctest_shim/ (doctest is not in this
#                image)
#   roster       prints the roster detect_backends() built (roster.cpp)
# The one registration line is applied to a copy of proj/src/lookup.cpp in
# baseline/accept/src/ (never committed): after `found` is declared in
# detect_backends(), the cuda entry goes first when a device answers, so the
# roster stays widest-first and scalar stays last (test_lookup.cpp:38-42).
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
REF=${REF:-/root/reference/proj}
OUT=$ROOT/baseline/accept
JSON=${JSON:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}
if [ ! -f "$REF/src/lookup.cpp" ]; then echo "reference checkout not present: nothing to build"; exit 0; fi
mkdir -p "$OUT/src" "$OUT/obj"
sed -e 's|#include "lookup_backend_detail.hpp"|#include "lookup_backend_detail.hpp"\nnamespace utf8v::detail { const lookup_backend\& cuda_backend(); bool cuda_available(); }|' \
    -e '/std::vector<lookup_backend> found;/a\  if (detail::cuda_available()) found.push_back(detail::cuda_backend());  // lookup_cuda.cpp' \
    "$REF/src/lookup.cpp" > "$OUT/src/lookup.cpp"
grep -q "cuda_available()) found.push_back" "$OUT/src/lookup.cpp"
CXX=${CXX:-g++}
FLAGS="-O3 -std=c++20 -DUTF8V_X86=1 -pthread -I$REF/include -I$REF/src -I$ROOT/include -I$JSON"
objs=()
build() {  # src obj [extra flags]
  local src=$1 obj=$OUT/obj/$2.o; shift 2
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then $CXX $FLAGS "$@" -c "$src" -o "$obj"; fi
  objs+=("$obj")
}
for f in oracle tables scalar fsm corpus bench lookup_scalar; do build "$REF/src/$f.cpp" "$f"; done
build "$REF/src/lookup_ssse3.cpp" lookup_ssse3 -mssse3
build "$REF/src/lookup_avx2.cpp" lookup_avx2 -mavx2
build "$OUT/src/lookup.cpp" lookup_registered
build "$ROOT/integration/reference_backend/lookup_cuda.cpp" lookup_cuda
LINK=(-L"$ROOT/paper_2010_03090_b200" -lutf8v_cuda -Wl,-rpath,'$ORIGIN/../../paper_2010_03090_b200' -pthread)
$CXX $FLAGS -o "$OUT/acceptance" "$REF/tests/acceptance.cpp" "${objs[@]}" "${LINK[@]}"
$CXX $FLAGS -I"$ROOT/integration/reference_backend/doctest_shim" -o "$OUT/unit_tests" \
    "$REF/tests/doctest_main.cpp" "$REF/tests/test_lookup.cpp" "$REF/tests/test_oracle.cpp" \
    "$REF/tests/test_tables.cpp" "${objs[@]}" "${LINK[@]}"
$CXX $FLAGS -o "$OUT/roster" "$ROOT/integration/reference_backend/roster.cpp" "${objs[@]}" "${LINK[@]}"
echo "built $OUT/acceptance $OUT/unit_tests $OUT/roster"
