#!/usr/bin/env bash
# Round-2 iteration call: bucket-sieve parity first, then the GPU suite,
# quick benches (1e12, 1e13, C5 window) and the cold-open breakdown.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_bucket.py -x -q > $O/pytest_bucket.txt 2>&1; echo "rc=$?" >> $O/pytest_bucket.txt
if [ "${FULL:-1}" = 1 ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
fi
for L in ${LIMITS:-1e12 1e13}; do
  GB_DEBUG_OPEN=1 timeout 300 python tools/quick_bench.py $L >> $O/qb.txt 2>&1
done
if [ "${C5:-1}" = 1 ]; then
  GB_DEBUG_OPEN=1 timeout 300 python tools/range_bench.py 4e18 1e11 2 > $O/c5.txt 2>&1
fi
ls -la $O
