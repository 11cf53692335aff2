#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for r in 1 2; do
for V in default m6_320k; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  echo "== $V 1e12 rep $r" >> $O/abm6.txt
  env $E timeout 200 python tools/quick_bench.py 1e12 2>&1 | grep -E "time=" | cut -c1-40 >> $O/abm6.txt
  echo "== $V C5 rep $r" >> $O/abm6.txt
  env $E timeout 200 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c44-60 >> $O/abm6.txt
done
done
