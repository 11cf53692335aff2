#!/usr/bin/env bash
# Round-2 measurement call: bench lines (C3, C4), C5 variants, ncu launch
# lists and full captures of the fused kernel at 1e12 and 1e13.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,persistence_mode --format=csv > $O/nvsmi.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_1e12.json 2> $O/bench_1e12.err
timeout 900 python bench.py --limit 1e13 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_1e13.json 2> $O/bench_1e13.err
c5() { echo "== $*" >> $O/c5var.txt; env "$@" timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep -E "time=|kernel" | cut -c1-140 >> $O/c5var.txt; }
c5 GB_SW=12
for V in ls4 ls1; do c5 GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so; done
if [ "${SKIP_NCU:-0}" != 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --limit 1e11 --steps 1 --warmup 3 --no-cpu-baseline --no-cli > $O/launches_bench.log 2>&1
for L in 1e12 1e13; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o $O/prof_verify_$L -f python tools/profile_one.py $L 9 > $O/ncu_full_$L.log 2>&1
done
fi
ls -la $O
