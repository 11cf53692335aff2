#!/usr/bin/env bash
# Session-3 closing call (after the deep-queue, scan-bound and split changes): GPU suite,
# smoke, bench lines, C2/C5 timings, launch list, ncu captures.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,persistence_mode --format=csv > $O/j_nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/j_pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/j_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/j_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/j_smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/j_bench_1e12.json 2> $O/j_bench_1e12.err
timeout 900 python bench.py --limit 1e13 --steps 3 --warmup 3 --no-cpu-baseline > $O/j_bench_1e13.json 2> $O/j_bench_1e13.err
timeout 300 python tools/range_bench.py 4e18 1e11 3 > $O/j_c5.txt 2>&1
timeout 300 python tools/quick_bench.py 1e10 > $O/j_c2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/j_launches_bench.csv \
  python bench.py --limit 1e11 --steps 1 --warmup 3 --no-cpu-baseline --no-cli > $O/j_launches_bench.log 2>&1
for L in 1e12 1e13; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o $O/j_proj_verify_$L -f python tools/profile_one.py $L 9 > $O/j_ncu_full_$L.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_large_rows -c 2 \
  -o $O/j_proj_large -f python tools/profile_one.py 4000000003200000000 8 > $O/j_ncu_large.log 2>&1
ls -la $O
