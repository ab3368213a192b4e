#!/bin/bash
# build/variants/<name>/libdk.so: libdk.so with extra nvcc flags for dk_kernels.cu (experiments)
# usage: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/paper_1510_02148_b200/_lib/obj
OUT=$ROOT/build/variants/$1
mkdir -p "$OUT"
/usr/local/cuda/bin/nvcc -c "$ROOT/paper_1510_02148_b200/csrc/dk_kernels.cu" -o "$OUT/dk_kernels.o" -O3 -std=c++17 \
  -Xcompiler -fPIC -I "$ROOT/include" -gencode arch=compute_100a,code=sm_100a -lineinfo $2
objs=$(ls $OBJ/*.o | grep -v dk_kernels.o)
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT/libdk.so" "$OUT/dk_kernels.o" $objs -cudart static
echo "$OUT/libdk.so"
