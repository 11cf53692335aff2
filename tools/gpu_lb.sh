#!/usr/bin/env bash
# k_large_batch (batch walk of the sparse large primes): thresholds on the C5
# window, launch list, C5 records and the large-prime tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for T in ${TS:-0 16777216 33554432 67108864 134217728 268435456}; do
  echo "== GB_LB_T=$T" >> $O/lb_c5.txt
  GB_LB_T=$T timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|kernel" | cut -c1-330 >> $O/lb_c5.txt
done
GB_LB_T=${NCU_T:-67108864} timeout 600 ncu -k regex:"k_large|k_verify_ws" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,sm__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file $O/lb_ncu.csv python tools/range_bench.py 4e18 1.6e10 1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_bigranges.py tests/test_gpu_bucket.py tests/test_gpu_edges.py -x -q > $O/lb_pytest.txt 2>&1; echo "rc=$?" >> $O/lb_pytest.txt
