#!/usr/bin/env bash
# GPU suite on the current build, then the sieve/check split at 1e12 / 1e13.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/s_pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/s_pytest_gpu.txt
for V in "GB_SW=12" "GB_SW=10" "GB_SW=16"; do
  for L in 1e12 1e13; do echo "== $V $L" >> $O/s_sw.txt; env $V timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/s_sw.txt; done
done
