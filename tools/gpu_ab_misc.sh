#!/usr/bin/env bash
# Split at 1e13 after the sieve-side cuts; warp-cooperative prime bound.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in "GB_SW=12" "GB_SW=10" "GB_SW=16"; do echo "== $V 1e13" >> $O/misc.txt; env $V timeout 300 python tools/quick_bench.py 1e13 2>&1 | grep -E "time=" | cut -c1-110 >> $O/misc.txt; done
for V in pw1536 pw2560; do
  for L in 1e12 1e13; do echo "== $V $L" >> $O/misc.txt; GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | cut -c1-110 >> $O/misc.txt; done
done
echo "== default 1e12" >> $O/misc.txt; timeout 300 python tools/quick_bench.py 1e12 2>&1 | grep -E "time=" | cut -c1-110 >> $O/misc.txt
