#!/usr/bin/env bash
# Session-3 baseline at HEAD: quick timings, C5 window, large-strike launch list, GPU suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,persistence_mode --format=csv > $O/base_smi.txt
for L in 1e12 1e13; do echo "== $L" >> $O/base_quick.txt; timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=|kernel" | cut -c1-160 >> $O/base_quick.txt; done
timeout 300 python tools/range_bench.py 4e18 1e11 3 > $O/base_c5.txt 2>&1
timeout 600 ncu -k regex:"k_large|k_verify_ws|k_segment" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,sm__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/base_c5_ncu.csv python tools/range_bench.py 4e18 3.2e9 1 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/base_pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/base_pytest_gpu.txt
