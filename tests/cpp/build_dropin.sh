#!/usr/bin/env bash
# Test infrastructure: links the reference's own AMR layer -- the UNCHANGED
# proj/src/{amr,macro_mesh,mesh_io,problems}.cpp, compiled from where they lie
# under /root/reference (no copies in this repository) -- against the B200
# facade: include/klref_b200/dropin comes first on the include path, so the
# hot-path headers klref/{hhg,fem,multigrid,estimator}.hpp are the facade's.
# Output: build/dropin/dropin_kl (git-ignored; travels to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REPO="$(cd "$HERE/../.." && pwd)"
REF="${KLREF_REFERENCE:-/root/reference}/proj"
OUT="$REPO/build/dropin"
if [ ! -d "$REF/src" ]; then
  echo "build_dropin: no reference sources at $REF (skipped)" >&2
  exit 0
fi
mkdir -p "$OUT"
SRCS=("$HERE/dropin_kl.cpp" "$REF/src/amr.cpp" "$REF/src/macro_mesh.cpp" "$REF/src/mesh_io.cpp" "$REF/src/problems.cpp")
newest=0
for f in "${SRCS[@]}" "$REPO"/include/klref_b200/klref.hpp "$REPO"/include/klref_b200.h "$REPO"/paper_2508_06049_b200/libklref_b200.so; do
  t=$(stat -c %Y "$f"); [ "$t" -gt "$newest" ] && newest=$t
done
if [ -x "$OUT/dropin_kl" ] && [ "$(stat -c %Y "$OUT/dropin_kl")" -ge "$newest" ]; then exit 0; fi
g++ -O2 -std=c++20 -Wall -Wno-unused-parameter \
  -I"$REPO/include/klref_b200/dropin" -I"$REPO/include" -I"$REF/include" \
  "${SRCS[@]}" -L"$REPO/paper_2508_06049_b200" -lklref_b200 \
  -Wl,-rpath,"\$ORIGIN/../../paper_2508_06049_b200" -o "$OUT/dropin_kl"
echo "built $OUT/dropin_kl"
