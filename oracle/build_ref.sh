#!/usr/bin/env bash
# Builds the UNMODIFIED-except-for-one-documented-patch reference library (arXiv 2604.15765,
# /root/reference/proj/src) plus our C-ABI shim (oracle/ref_capi.cpp) into oracle/_ref/.
#
# TEST INFRASTRUCTURE ONLY: the product never links or loads anything built here.
#
#  * The reference sources are compiled where they lie under /root/reference (never copied
#    into the repo).  The single exception is proj/src/kernels.cpp, of which a patched copy
#    is written to oracle/_ref/gen/ (git-ignored) with three index swaps at kernels.cpp:365,
#    :367, :369 (tiled_two_mixed writes wrong hermitian mirrors on
#    diagonal base pairs).  An unpatched build is produced as well, to document the bug.
#  * CMake is not used: proj/CMakeLists.txt:16-18 adds src/, tools/, tests/ which do not exist.
#  * Flags: the paper's -O3 -fno-strict-aliasing; -march=x86-64-v3 instead of
#    -march=native so the .so also runs on a GPU box whose host CPU differs from this one.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${HERMSIM_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: $REF not present; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT/gen" "$OUT/obj" "$OUT/obj_unpatched"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O3 -march=x86-64-v3 -fno-strict-aliasing -fPIC -pthread -w -I$REF/include"

# patched copy of kernels.cpp (three mirror-index swaps)
sed -e '365s/idx(0, ci, 0, ri)/idx(0, ri, 0, ci)/' \
    -e '367s/idx(1, ci, 1, ri)/idx(1, ri, 1, ci)/' \
    -e '369s/idx(0, ci, 1, ri)/idx(0, ri, 1, ci)/' "$REF/src/kernels.cpp" > "$OUT/gen/kernels_patched.cpp"
if cmp -s "$REF/src/kernels.cpp" "$OUT/gen/kernels_patched.cpp"; then
  echo "build_ref: patch did not apply" >&2; exit 1
fi
[ "$(diff "$REF/src/kernels.cpp" "$OUT/gen/kernels_patched.cpp" | grep -c '^<')" = 3 ] || { echo "build_ref: unexpected patch size" >&2; exit 1; }

pids=()
for f in channel linalg native parallel storage storage_io; do
  $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" & pids+=($!)
done
$CXX $FLAGS -c "$OUT/gen/kernels_patched.cpp" -o "$OUT/obj/kernels.o" & pids+=($!)
$CXX $FLAGS -c "$REF/src/kernels.cpp" -o "$OUT/obj_unpatched/kernels.o" & pids+=($!)
$CXX $FLAGS -c "$HERE/ref_capi.cpp" -o "$OUT/obj/ref_capi.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done

COMMON="$OUT/obj/channel.o $OUT/obj/linalg.o $OUT/obj/native.o $OUT/obj/parallel.o $OUT/obj/storage.o $OUT/obj/storage_io.o $OUT/obj/ref_capi.o"
$CXX -shared -pthread -o "$OUT/libhermsim_ref.so" $COMMON "$OUT/obj/kernels.o"
$CXX -shared -pthread -o "$OUT/libhermsim_ref_unpatched.so" $COMMON "$OUT/obj_unpatched/kernels.o"
echo "build_ref: built $OUT/libhermsim_ref.so and libhermsim_ref_unpatched.so"
