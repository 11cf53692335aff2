# ncu full capture of one fused launch (top segments below LIM) + its source page
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for LIM in ${LIMS:-1e12}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o gpurun_out/prof_verify_$LIM -f python tools/profile_one.py $LIM 9 > gpurun_out/ncu_full_$LIM.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$LIM.log
done
