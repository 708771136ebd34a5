#!/bin/bash
# A/B build: tools/build_variant.sh NAME "-DFLAG=..." [changed .cu files]  ->  paper_1607_08220_b200/libkdtree_NAME.so
# (only the listed translation units are recompiled with the extra flags; select it with KDB_LIB_PATH)
set -e
NAME=$1; FLAGS=$2; shift 2
SRCS=${@:-kd_build_f32.cu kd_build_f64.cu}
cd "$(dirname "$0")/../paper_1607_08220_b200/csrc"
make -s -j4 >/dev/null 2>&1
mkdir -p build_$NAME
OBJS=""
for f in kd_build_f32.cu kd_build_f64.cu kd_query.cu kd_walk.cu kd_packet.cu kd_capi.cu kd_dist.cu; do
  if [[ " $SRCS " == *" $f "* ]]; then
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $FLAGS -c $f -o build_$NAME/${f%.cu}.o &
    OBJS="$OBJS build_$NAME/${f%.cu}.o"
  else
    OBJS="$OBJS build/${f%.cu}.o"
  fi
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libkdtree_$NAME.so $OBJS -Xcompiler -fPIC
echo built ../libkdtree_$NAME.so
