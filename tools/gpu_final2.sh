#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,persistence_mode --format=csv > $O/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_1e12.json 2> $O/bench_1e12.err
timeout 900 python bench.py --limit 1e13 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_1e13.json 2> $O/bench_1e13.err
timeout 300 python tools/range_bench.py 4e18 1e11 3 > $O/c5_final.txt 2>&1
timeout 300 python tools/quick_bench.py 1e10 > $O/c2_final.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --limit 1e11 --steps 1 --warmup 3 --no-cpu-baseline --no-cli > $O/launches_bench.log 2>&1
for L in 1e12 1e13; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o $O/prof_verify_$L -f python tools/profile_one.py $L 9 > $O/ncu_full_$L.log 2>&1
done
ls -la $O
