#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for L in 1e13 1e12; do
  echo "== skipsingle $L (wrong results, timing probe)" >> $O/probe.txt
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/skipsingle/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | tail -1 | cut -c1-60 >> $O/probe.txt
  echo "== skipsingle $L GB_SW=12" >> $O/probe.txt
  GB_SW=12 GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/skipsingle/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | tail -1 | cut -c1-60 >> $O/probe.txt
done
