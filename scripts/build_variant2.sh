#!/bin/bash
# Like build_variant.sh with several sources recompiled under the same -D flags:
# bash scripts/build_variant2.sh NAME "-DFOO=1" SRC1 SRC2 ... -> _variants/NAME.so
set -e
NAME=$1; DEFS=$2; shift 2
cd "$(dirname "$0")/.."
python -c "from paper_2407_17437_b200 import build; build.build()"
mkdir -p build/var _variants
EXCL=""; NEW=""
for SRC in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include $DEFS \
    -c paper_2407_17437_b200/csrc/$SRC.cu -o build/var/${NAME}_$SRC.o
  EXCL="$EXCL|/$SRC.o\$"; NEW="$NEW build/var/${NAME}_$SRC.o"
done
OBJS=$(ls build/csrc/*.o | grep -v -E "${EXCL:1}")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$NAME.so $OBJS $NEW
