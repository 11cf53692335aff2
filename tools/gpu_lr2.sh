#!/usr/bin/env bash
# k_large_rows with the fused first index and streaming loads; coprime-skip
# levels 0/1/2 against the per-slot rows on the C5 window; parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in "GB_LS_ROWS=0" "GB_LS_COP=0" "GB_LS_COP=1" "GB_LS_COP=2"; do
  echo "== $V" >> $O/lr2_c5.txt
  env $V timeout 300 python tools/range_bench.py 4e18 1e11 3 2>&1 | grep -E "time=|kernel" | cut -c1-330 >> $O/lr2_c5.txt
done
for V in "GB_LS_COP=1" "GB_LS_COP=2"; do
env $V timeout 600 ncu -k regex:"k_large|k_verify_ws" \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,sm__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none --csv --log-file "$O/lr2_ncu_${V#*=}.csv" python tools/range_bench.py 4e18 1.6e10 1 > /dev/null 2>&1
done
timeout 900 python -m pytest tests/test_gpu_bigranges.py tests/test_gpu_bucket.py tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q > $O/lr2_pytest.txt 2>&1; echo "rc=$?" >> $O/lr2_pytest.txt
GB_LS_COP=2 timeout 900 python -m pytest tests/test_gpu_bigranges.py -k c5 -x -q >> $O/lr2_pytest.txt 2>&1; echo "cop2 rc=$?" >> $O/lr2_pytest.txt
