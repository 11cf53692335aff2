#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for L in 1e12 1e13; do
  echo "== pair(group wait) $L" >> $O/pair2.txt
  GB_PAIR=1 timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | tail -1 | cut -c1-150 >> $O/pair2.txt
  echo "== pair noremote probe $L" >> $O/pair2.txt
  GB_PAIR=1 GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/noremote/libgoldbach_b200.so timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | tail -1 | cut -c1-60 >> $O/pair2.txt
done
