#!/usr/bin/env bash
# run-loop strikes with IMAD addressing (runimad) against the default.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for R in 1 2; do for V in default runimad; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e13; do echo "== $V $L" >> $O/runab.txt; env $E timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/runab.txt; done
done; done
