#!/usr/bin/env bash
# C5-window variants: large-strike slot grouping, mask fill on/off, rows in flight
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
run() { echo "== $*" >> $O/c5var.txt; env "$@" timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|kernel" | cut -c1-120 >> $O/c5var.txt; }
run GB_MASK_P=0
run GB_MASK_P=262145
for V in ${VARIANTS:-ls4 ls1 mk8}; do
  run GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so GB_MASK_P=262145
done
