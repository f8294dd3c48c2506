#!/bin/bash
# A/B experiments: rebuild one CUDA source with extra flags into a separate
# library under variants/ (git-ignored), then select it with SGTK_LIB.
#   bash tools/build_variant.sh <name> <source stem> [-DFLAG=...]
#   SGTK_LIB=$PWD/variants/libsgtk_<name>.so python tools/agnn_only.py
set -e
name=$1; stem=$2; shift 2
cd "$(dirname "$0")/../paper_2412_12218_b200/csrc"
make -s -j16 >/dev/null
mkdir -p ../../variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -ccbin /usr/bin/g++ -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -I../../include -I. \
  --expt-relaxed-constexpr "$@" -c $stem.cu -o build/${stem}_variant.o
objs=$(ls build/*.o | grep -v "build/${stem}.o\|_variant.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ \
  -o ../../variants/libsgtk_$name.so $objs build/${stem}_variant.o -Xlinker --exclude-libs,ALL
rm build/${stem}_variant.o
echo "variants/libsgtk_$name.so"
