#!/bin/bash
# A/B build of the library with extra macros into build_ab/<name>.so (objects in build_ab/<name>/).
#   bash tools/build_variant.sh NAME "-DAM_FOO=1 -DAM_BAR=2"
set -e
NAME=$1; EXTRA=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2004_00540_b200/csrc
OUT=$ROOT/build_ab/$NAME
mkdir -p "$OUT"
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -ccbin g++ -I$ROOT/include $EXTRA"
pids=()
for f in stencil bits trace capi multigpu batch mapio upload; do
  $NVCC $FLAGS -c $SRC/$f.cu -o $OUT/$f.o & pids+=($!)
done
for f in actmap_api report pack; do
  g++ -std=c++20 -O2 -fPIC -I$ROOT/include -c $SRC/$f.cpp -o $OUT/$f.o & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
$NVCC $ARCH -shared -cudart static -o $ROOT/build_ab/$NAME.so $OUT/*.o -ldl -lpthread
rm -rf "$OUT"
echo "built build_ab/$NAME.so"
