# launch list of the large-strike kernel (C5 window) per variant in build/variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in ${VARS:-ls4}; do
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$v/libgoldbach_b200.so timeout 600 ncu -k regex:k_large_strike \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_op_red.sum,sm__inst_executed.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --csv --log-file gpurun_out/large_$v.csv python tools/range_bench.py ${START:-4e18} ${SPAN:-1e10} 1 > /dev/null 2>&1
done
