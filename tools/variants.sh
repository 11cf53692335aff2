#!/usr/bin/env bash
# Build kernel variants for an A/B timing run on the GPU:
#   tools/variants.sh NAME "GEN_ARGS" "EXTRA_NVFLAGS" [NAME "GEN_ARGS" "EXTRA_NVFLAGS" ...]
# Each variant lands in build/variants/NAME/libgoldbach_b200.so; the in-tree
# header and library are rebuilt with the defaults afterwards.
# Time them with: GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/NAME/libgoldbach_b200.so python tools/quick_bench.py 1e12
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 3 ]; do
  name=$1; gen=$2; nv=$3; shift 3
  python tools/gen_bitslice.py $gen > /dev/null
  touch paper_2603_07850_b200/csrc/gb_kernels.cu
  make -s -j16 NVEXTRA="$nv" paper_2603_07850_b200/libgoldbach_b200.so 2>&1 | grep -E "error" || true
  mkdir -p build/variants/$name
  cp paper_2603_07850_b200/libgoldbach_b200.so build/variants/$name/
  echo "built $name"
done
python tools/gen_bitslice.py > /dev/null
touch paper_2603_07850_b200/csrc/gb_kernels.cu
make -s -j16 2>&1 | grep -E "error" || true
