#!/usr/bin/env bash
# Same-box A/B: first-index chain off (no stream waits) / on; sieve/check
# split at the C5 height; ncu capture of the fused kernel at C5 height.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in "GB_LS_CHAIN=0" "GB_LS_CHAIN=1" "GB_LS_CHAIN=0" "GB_LS_CHAIN=1" "GB_SW=10" "GB_SW=16"; do
  echo "== $V" >> $O/chain2_c5.txt
  env $V timeout 300 python tools/range_bench.py 4e18 1e11 3 2>&1 | grep -E "time=|kernel" | cut -c1-330 >> $O/chain2_c5.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o $O/f_prof_verify_c5 -f python tools/profile_one.py 4000000003600000000 9 > $O/f_ncu_full_c5.log 2>&1
