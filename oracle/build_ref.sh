#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Builds the UNMODIFIED reference implementation from its own
# sources where they lie (/root/reference/proj/src/*.cpp) with the reference's own Release
# flags (-std=c++20 -O3 -DNDEBUG, no -march; proj/CMakeLists.txt:8-10, src/CMakeLists.txt:18),
# namespace-renamed to sht_ref (-Dsht=sht_ref) so it can share a process with the drop-in,
# plus the C shim oracle/ref_shim.cpp.  Output goes only to oracle/_ref/ (git-ignored, but it
# travels to the GPU box with gpurun so the oracle and the CPU baseline exist there).
# The reference's own CMake build is not used.  Reference sources are never copied.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${SHT_REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference sources not found at $REF (prebuilt oracle/_ref is used as-is)" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -Dsht=sht_ref -I$REF/include"
objs=()
for src in "$REF"/src/*.cpp "$HERE/ref_shim.cpp"; do
  obj="$OUT/obj/$(basename "${src%.cpp}").o"
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then
    $CXX $FLAGS -c "$src" -o "$obj" &
  fi
  objs+=("$obj")
done
wait
$CXX -shared -o "$OUT/libsht_ref.so.tmp" "${objs[@]}" -lpthread
mv "$OUT/libsht_ref.so.tmp" "$OUT/libsht_ref.so"
# static archive of the reference alone (for C++ parity binaries that link sht_ref:: directly)
ar rcs "$OUT/libsht_ref_core.a.tmp" $(ls "$OUT"/obj/*.o | grep -v ref_shim.o)
mv "$OUT/libsht_ref_core.a.tmp" "$OUT/libsht_ref_core.a"
echo "build_ref: $OUT/libsht_ref.so"
