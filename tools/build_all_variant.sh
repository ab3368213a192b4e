#!/bin/bash
# build/variants/<name>/libdk.so: every source compiled with extra nvcc flags (experiments,
# e.g. the timeline build: tools/build_all_variant.sh tl -DDK_TIMELINE)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/variants/$1
mkdir -p "$OUT"
SRCS="dk_device dk_kernels dk_coarse dk_dense dk_profile dk_setup dk_api"
for s in $SRCS; do
  /usr/local/cuda/bin/nvcc -c "$ROOT/paper_1510_02148_b200/csrc/$s.cu" -o "$OUT/$s.o" -O3 -std=c++17 \
    -Xcompiler -fPIC -I "$ROOT/include" -gencode arch=compute_100a,code=sm_100a -lineinfo $2 &
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT/libdk.so" \
  $(for s in $SRCS; do echo "$OUT/$s.o"; done) -cudart static
rm -f "$OUT"/*.o
echo "$OUT/libdk.so"
