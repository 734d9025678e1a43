# Builds diagnostic variants of the library (D=3, m=2 only) for GPU A/B runs:
#   scripts/build_variants.sh name "-DFLAG=1 ..." [name2 "flags2" ...]
# -> build_variants/lib<name>.so ; select with SPHRAY_B200_LIB at run time.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -C "$ROOT/paper_2401_02896_b200/csrc" -j16 OUT="$ROOT/build_variants/lib$name.so" \
       OBJ="$ROOT/build_variants/obj_$name" EXTRA_NVFLAGS="-DSPHRAY_FAST_BUILD $flags" EXTRA_CXXFLAGS="$flags" >/dev/null
  echo "built build_variants/lib$name.so ($flags)"
done
