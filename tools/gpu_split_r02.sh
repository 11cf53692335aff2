#!/usr/bin/env bash
# Mask fill + split variants at 1e12 / 1e13 / C5, cold-open breakdown, CLI process time.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
q() { echo "== $*" >> $O/split.txt; env "$@" timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=|kernel" | cut -c1-140 >> $O/split.txt; }
for L in 1e13 1e12; do
  q GB_MASK_P=0
  q GB_MASK_P=262145
  q GB_MASK_P=262145 GB_SW=12
  q GB_MASK_P=524288
  q GB_MASK_P=1048576 GB_SW=10
done
echo "== C5" >> $O/split.txt
for M in 0 262145; do for S in 10 12 16; do
  echo "== C5 GB_MASK_P=$M GB_SW=$S" >> $O/split.txt
  GB_MASK_P=$M GB_SW=$S timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|kernel" | cut -c1-120 >> $O/split.txt
done; done
GB_DEBUG_OPEN=1 timeout 300 python tools/open_probe.py > $O/open.txt 2>&1
for i in 1 2 3; do /usr/bin/time -f "cli wall %e s" ./paper_2603_07850_b200/bin/goldbach 1000000000000 --gpus=1 --json >> $O/open.txt 2>&1; done
GB_DEBUG_OPEN=1 ./paper_2603_07850_b200/bin/goldbach 1000000000000 --gpus=1 --json >> $O/open.txt 2>&1
