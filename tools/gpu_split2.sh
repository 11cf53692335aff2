#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
q() { L=$1; shift; echo "== $L $*" >> $O/split2.txt; env "$@" timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | tail -1 | cut -c1-40 >> $O/split2.txt; }
q 1e12 GB_SW=10; q 1e12 GB_SW=12; q 1e12 GB_SW=16
q 1e13 GB_SW=12; q 1e13 GB_SW=16; q 1e13 GB_SW=10
for S in 10 12 16; do echo "== C5 GB_SW=$S" >> $O/split2.txt; GB_SW=$S timeout 200 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | tail -1 | cut -c44-60 >> $O/split2.txt; done
