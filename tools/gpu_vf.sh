#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in default vf20 vf24; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e13; do
    echo "== $V $L" >> $O/vf.txt
    env $E timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | tail -1 | cut -c1-40 >> $O/vf.txt
  done
done
