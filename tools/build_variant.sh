#!/bin/bash
# Build a variant of libkle_b200.so with one source recompiled under extra flags.
# usage: tools/build_variant.sh NAME SOURCE.cu "-DFOO=1 ..."   -> paper_2510_26180_b200/lib/variants/libkle_NAME.so
set -e
cd "$(dirname "$0")/../paper_2510_26180_b200/csrc"
make -s >/dev/null
NAME=$1; SRC=$2; FLAGS=$3
mkdir -p build/var_$NAME ../lib/variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -Xptxas -v $FLAGS -c $SRC -o build/var_$NAME/${SRC%.cu}.o 2> build/var_$NAME/ptxas.log
OBJS=""
for o in build/*.o; do b=$(basename $o); if [ "$b" == "${SRC%.cu}.o" ]; then OBJS="$OBJS build/var_$NAME/$b"; else OBJS="$OBJS $o"; fi; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../lib/variants/libkle_$NAME.so $OBJS
echo built ../lib/variants/libkle_$NAME.so
