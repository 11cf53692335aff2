#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
python tools/cli_timing.py 1e12 1 3 > $O/cli_timing2.txt 2>&1
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
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/quick_bench.py 1e13 2>&1 | grep -E "time=" | cut -c1-100 >> $O/bounds.txt
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/quick_bench.py 1e12 2>&1 | grep -E "time=" | cut -c1-100 >> $O/bounds.txt
done
timeout ${GOLD_SECS:-1800} python oracle/make_big_goldens.py --set c4 --part ${GOLD_PART:-0:5000} --jobs 16 --skip oracle/_ref/c4_done.tsv \
  --out $O/c4_part.tsv > $O/c4_gen_part.log 2>&1
wc -l $O/c4_part.tsv
