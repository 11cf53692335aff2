#!/usr/bin/env bash
# Per-class scan bounds after the word-entry deep queue (variants from
# tools/variants.sh) at 1e12 / 1e13 / C5, plus GB_SW=16 at 1e13.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in ${VARS:-default b227_449 b227_503 b257_449 b293_557}; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e13; do echo "== $V $L" >> $O/${OUT:-bab}.txt; env $E timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/${OUT:-bab}.txt; done
  echo "== $V C5" >> $O/${OUT:-bab}.txt; env $E timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c1-200 >> $O/${OUT:-bab}.txt
done
if [ -z "$NOSW" ]; then
echo "== GB_SW=16 1e13" >> $O/${OUT:-bab}.txt; GB_SW=16 timeout 300 python tools/quick_bench.py 1e13 2>&1 | grep -E "time=" | cut -c1-110 >> $O/${OUT:-bab}.txt
echo "== GB_SW=10 C5" >> $O/${OUT:-bab}.txt; GB_SW=10 timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c1-200 >> $O/${OUT:-bab}.txt
fi
