#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
S=compute-sanitizer
( timeout 900 $S --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
  for m in rows mask large; do
    echo "== racecheck $m"; timeout 900 $S --tool racecheck --racecheck-report hazard python tools/sanitize_r02.py $m 2>&1 | tail -3
    echo "== memcheck $m"; timeout 900 $S --tool memcheck python tools/sanitize_r02.py $m 2>&1 | tail -2
  done
  echo "== racecheck pair"; GB_PAIR=1 timeout 900 $S --tool racecheck --racecheck-report hazard python tools/sanitize_r02.py rows 2>&1 | tail -3
) > $O/sanitizer2.txt 2>&1
for L in 1e12 1e13; do GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/stats/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "stats|time=" | tail -2 >> $O/stats2.txt; done
GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/stats/libgoldbach_b200.so timeout 300 python - >> $O/stats2.txt 2>&1 <<'PY'
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
