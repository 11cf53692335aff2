#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
GB_PAIR=1 GB_DEBUG_OPEN=1 timeout 120 python tools/quick_bench.py 1e10 > $O/pair.txt 2>&1; echo "rc=$?" >> $O/pair.txt
for L in 1e12 1e13; do
  echo "== pair $L" >> $O/pair.txt
  GB_PAIR=1 timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | cut -c1-200 >> $O/pair.txt
  echo "== pair $L SW=12" >> $O/pair.txt
  GB_PAIR=1 GB_SW=12 timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror" | cut -c1-200 >> $O/pair.txt
done
echo "== pair C5" >> $O/pair.txt
GB_PAIR=1 timeout 200 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|rror" | cut -c1-200 >> $O/pair.txt
GB_PAIR=1 timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py tests/test_gpu_wheel.py -x -q > $O/pytest_pair.txt 2>&1; echo rc=$? >> $O/pytest_pair.txt
