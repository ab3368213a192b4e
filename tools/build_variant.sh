#!/bin/bash
# build/variants/<name>/libdk.so: libdk.so with extra nvcc flags for one source (experiments)
# usage: tools/build_variant.sh NAME "-DFOO=1 ..." [SOURCE_STEM (default dk_kernels)]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_1510_02148_b200/_lib/obj
SRC=${3:-dk_kernels}
OUT=$ROOT/build/variants/$1
mkdir -p "$OUT"
/usr/local/cuda/bin/nvcc -c "$ROOT/paper_1510_02148_b200/csrc/$SRC.cu" -o "$OUT/$SRC.o" -O3 -std=c++17 \
  -Xcompiler -fPIC -I "$ROOT/include" -gencode arch=compute_100a,code=sm_100a -lineinfo $2
objs=$(ls $OBJ/*.o | grep -v "/$SRC.o")
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT/libdk.so" "$OUT/$SRC.o" $objs -cudart static
echo "$OUT/libdk.so"
