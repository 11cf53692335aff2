#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
q() { echo "== $*" >> $O/more_var.txt; env "$@" timeout 300 python tools/quick_bench.py 1e13 2>&1 | grep -E "time=" | tail -1 | cut -c1-60 >> $O/more_var.txt; }
q GB_MASK_P=0
q GB_MASK_P=2097152 GB_SW=16
q GB_MASK_P=2097152 GB_SW=12
q GB_MASK_P=2621440 GB_SW=16
q GB_MASK_P=2621440 GB_SW=12
q GB_MASK_P=3000017 GB_SW=16
echo "== C5 ls4" >> $O/more_var.txt
GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/ls4/libgoldbach_b200.so timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | tail -1 | cut -c1-80 >> $O/more_var.txt
echo "== C5 default" >> $O/more_var.txt
timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | tail -1 | cut -c1-80 >> $O/more_var.txt
timeout 300 ./paper_2603_07850_b200/bin/ref_api_conformance --gpu >> $O/more_var.txt 2>&1
