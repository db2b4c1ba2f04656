#!/usr/bin/env bash
# Test infrastructure (oracle), not product code.
#
# Builds the *patched* reference hot path into oracle/_ref/ straight from the
# sources where they lie under /root/reference/proj (no copies are written):
# each translation unit is streamed through sed and compiled from stdin.
#
# Two one-line defects of the shipped reference are fixed on the fly
# (SURVEY.md §0.3); without them the reference hot path produces NaN / zero
# estimates, so "the reference" for parity means "reference + D1/D2":
#   D1  proj/src/fem.cpp:32      stiffness_matrix uses the signed area -> |area|
#   D2  proj/src/hhg.cpp:170-172 boundary_group ignores edge orientation ->
#       position along the edge counted from the lower-id corner, as the
#       groups are built at proj/src/hhg.cpp:114-123.
#
# Flags follow SURVEY.md §0.4: -std=c++20 -O2, no -march, no -ffast-math
# (x86-64 SSE2: no FMA contraction).  A second build with FMA contraction
# (-O3 -march=native -ffp-contract=fast) is produced as ref_driver_fma to
# report the reference's own rounding noise floor beside the parity numbers.
#
# Outputs: oracle/_ref/ref_driver, oracle/_ref/ref_driver_fma (git-ignored,
# but they travel to the GPU box with gpurun like the other built files).
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${KLREF_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref.sh: reference sources not found at $REF (skipping)" >&2
  exit 0
fi
mkdir -p "$OUT/obj" "$OUT/obj_fma"

SRCS="macro_mesh mesh_io hhg fem problems multigrid estimator amr"

# sed programs for the two fixes; each must match exactly once.
D1='s/const double area = 0\.5 \* area2;/const double area = 0.5 * std::fabs(area2);/'
POS0='(corner_ids_[static_cast<std::size_t>(slot)][0] < corner_ids_[static_cast<std::size_t>(slot)][1] ? i : n - i)'
POS1='(corner_ids_[static_cast<std::size_t>(slot)][0] < corner_ids_[static_cast<std::size_t>(slot)][2] ? j : n - j)'
POS2='(corner_ids_[static_cast<std::size_t>(slot)][1] < corner_ids_[static_cast<std::size_t>(slot)][2] ? j : n - j)'
D2A="s/if (j == 0) return ml\.edge\[0\]\.group_start + (i - 1);/if (j == 0) return ml.edge[0].group_start + ($POS0 - 1);/"
D2B="s/if (i == 0) return ml\.edge\[1\]\.group_start + (j - 1);/if (i == 0) return ml.edge[1].group_start + ($POS1 - 1);/"
D2C="s/if (i + j == n) return ml\.edge\[2\]\.group_start + (j - 1);/if (i + j == n) return ml.edge[2].group_start + ($POS2 - 1);/"

patched() {  # $1 = unit name; writes the patched source to stdout
  local f="$REF/src/$1.cpp"
  case "$1" in
    fem) sed -e "$D1" "$f" ;;
    hhg) sed -e "$D2A" -e "$D2B" -e "$D2C" "$f" ;;
    *) cat "$f" ;;
  esac
}

# verify the patches apply exactly once each
[ "$(patched fem | grep -c 'std::fabs(area2)')" = "1" ] || { echo "D1 patch failed" >&2; exit 1; }
[ "$(patched hhg | grep -c 'corner_ids_\[static_cast<std::size_t>(slot)\]\[.\] < corner_ids_')" = "3" ] || { echo "D2 patch failed" >&2; exit 1; }

CXX="${CXX:-g++}"
BASE_FLAGS="-std=c++20 -I$REF/include"
for u in $SRCS; do
  patched "$u" | $CXX $BASE_FLAGS -O2 -x c++ -c - -o "$OUT/obj/$u.o"
  patched "$u" | $CXX $BASE_FLAGS -O3 -march=native -ffp-contract=fast -x c++ -c - -o "$OUT/obj_fma/$u.o"
done
$CXX $BASE_FLAGS -O2 -c "$HERE/ref_driver.cpp" -o "$OUT/obj/ref_driver.o"
$CXX $BASE_FLAGS -O3 -march=native -ffp-contract=fast -c "$HERE/ref_driver.cpp" -o "$OUT/obj_fma/ref_driver.o"
# the builder's 3-d C oracle (config 4 AMR meshes: eta_T for the reference's 3-d refinement)
${CC:-gcc} -O2 -std=c11 -D_GNU_SOURCE -c "$HERE/klref_oracle3d.c" -o "$OUT/obj/oracle3d.o"
cp "$OUT/obj/oracle3d.o" "$OUT/obj_fma/oracle3d.o"
$CXX -o "$OUT/ref_driver" "$OUT"/obj/*.o -lm
$CXX -o "$OUT/ref_driver_fma" "$OUT"/obj_fma/*.o -lm
echo "built $OUT/ref_driver and $OUT/ref_driver_fma"
