#!/usr/bin/env bash
# 8 sieve warps (20 check warps) for the low-prime split at 1e12 against the default 10.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for R in 1 2; do for V in default m8; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e11; do echo "== $V $L" >> $O/m8.txt; env $E timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | cut -c1-110 >> $O/m8.txt; done
done; done
