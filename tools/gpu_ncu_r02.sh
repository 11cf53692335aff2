#!/usr/bin/env bash
# ncu: launch list + full captures of the bucket fill and the fused kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for L in ${LIMS:-1e13}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$L.csv \
  python tools/profile_one.py $L 8 > $O/launches_$L.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bucket_fill|k_verify_ws" -s ${SKIP:-0} -c 2 \
  -o $O/prof_$L -f python tools/profile_one.py $L 8 > $O/ncu_full_$L.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full_$L.log
done
ls -la $O
