#!/bin/bash
# Build a tuning variant of the library with one source recompiled under extra
# -D flags: bash scripts/build_variant.sh NAME SRC "-DFOO=1 -DBAR=2"
# -> _variants/NAME.so (load it with SMB_LIB=_variants/NAME.so)
set -e
NAME=$1; SRC=$2; DEFS=$3
cd "$(dirname "$0")/.."
python -c "from paper_2407_17437_b200 import build; build.build()"
mkdir -p build/var _variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --fmad=false \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I include $DEFS \
  -c paper_2407_17437_b200/csrc/$SRC.cu -o build/var/${NAME}_$SRC.o
OBJS=$(ls build/csrc/*.o | grep -v "/$SRC.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _variants/$NAME.so $OBJS build/var/${NAME}_$SRC.o
