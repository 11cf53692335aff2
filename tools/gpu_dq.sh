#!/usr/bin/env bash
# Word-entry deep queue (default) against the per-even queue (dq0): 1e12,
# 1e13, C5; then the GPU suite on the default build.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for R in 1 2; do
for V in default dq0; do
  if [ $V = default ]; then E=""; else E="GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so"; fi
  for L in 1e12 1e13; do echo "== $V $L" >> $O/dq.txt; env $E timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/dq.txt; done
  echo "== $V C5" >> $O/dq.txt; env $E timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c1-200 >> $O/dq.txt
done
done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/dq_pytest.txt 2>&1; echo "rc=$?" >> $O/dq_pytest.txt
