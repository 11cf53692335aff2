#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for E in "GB_LS_PRE=0" "GB_LS_PRE=1"; do
  echo "== $E" >> $O/c5pre.txt
  env $E timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|kernel" | cut -c1-160 >> $O/c5pre.txt
done
timeout 900 python -m pytest tests/test_gpu_bigranges.py tests/test_gpu_tile.py tests/test_gpu_parity.py -x -q -k "c5 or ceiling or large or 4000000" > $O/pytest_c5.txt 2>&1; echo rc=$? >> $O/pytest_c5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_large" -s 3 -c 2 \
  -o $O/prof_c5_pre -f python tools/profile_one.py 4000000100000000000 9 > $O/ncu_c5_pre.log 2>&1
