#!/bin/bash
# Build an A/B variant of the library: recompile ONE source with extra
# defines, link it with the in-tree objects into ab_lib/<name>.so.
#   tools/build_variant.sh minb6 gb_mv_binned.cu -DGB_MVB_MINB=6
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; SRC=$2; shift 2
C="$ROOT/paper_1908_01407_b200/csrc"
mkdir -p "$ROOT/ab_lib/obj_$NAME"
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I"$ROOT/include" "$@" \
  -c "$C/$SRC" -o "$ROOT/ab_lib/obj_$NAME/${SRC%.cu}.o"
OBJS=""
for o in "$C"/build/*.o; do
  b=$(basename "$o")
  if [ "$b" = "${SRC%.cu}.o" ]; then OBJS="$OBJS $ROOT/ab_lib/obj_$NAME/$b"; else OBJS="$OBJS $o"; fi
done
nvcc $ARCH -shared -o "$ROOT/ab_lib/$NAME.so" $OBJS -lcudart
echo "built ab_lib/$NAME.so"
