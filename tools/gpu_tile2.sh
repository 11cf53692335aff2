#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in ${VARS:-default}; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e13; do
    echo "== $V $L" >> $O/tile2.txt
    env $E timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|Error" | tail -1 | cut -c1-150 >> $O/tile2.txt
  done
  echo "== $V C5" >> $O/tile2.txt
  env $E timeout 200 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|Error" | tail -1 | cut -c1-70 >> $O/tile2.txt
done
