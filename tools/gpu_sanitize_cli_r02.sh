#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_bucket.py -x -q > $O/pytest_tile.txt 2>&1; echo rc=$? >> $O/pytest_tile.txt
python tools/cli_timing.py 1e12 1 3 > $O/cli_timing.txt 2>&1
python tools/cli_timing.py 1e10 1 2 >> $O/cli_timing.txt 2>&1
S=compute-sanitizer
( timeout 900 $S --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4
  for m in rows mask large; do
    echo "== racecheck $m"; timeout 900 $S --tool racecheck --racecheck-report hazard python tools/sanitize_r02.py $m 2>&1 | tail -4
    echo "== memcheck $m"; timeout 900 $S --tool memcheck python tools/sanitize_r02.py $m 2>&1 | tail -3
  done ) > $O/sanitizer.txt 2>&1
for L in 1e12 1e13; do GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/stats/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "stats|time=" | tail -2 >> $O/stats.txt; done
GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/stats/libgoldbach_b200.so timeout 300 python - >> $O/stats.txt 2>&1 <<'PY'
import sys, ctypes as C
sys.path.insert(0, '.')
import paper_2603_07850_b200 as gb
dev = gb.Device(4 * 10**18 + 10**11)
v = (C.c_uint64 * 8)(); gb.lib().gb_debug_stats(v, 1)
pool = gb.Pool(4 * 10**18, 4 * 10**18 + 10**11, 200_000_000)
r = gb.drain_pool(dev, pool)
gb.lib().gb_debug_stats(v, 1)
print("C5 stats [generic evens, inplace deep, queued deep, deep rounds, stragglers, fast blocks, generic blocks]:", list(v), r.as_dict()["evens"])
PY
for V in b383 b563 b383_563; do
  echo "== $V" >> $O/bounds.txt
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c1-100 >> $O/bounds.txt
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/quick_bench.py 1e12 2>&1 | grep -E "time=" | cut -c1-100 >> $O/bounds.txt
done
echo "== default" >> $O/bounds.txt
timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=" | cut -c1-100 >> $O/bounds.txt
