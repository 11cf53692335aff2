#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list and one
# full ncu capture of the fused kernel.  Outputs land in gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py --steps 3 --warmup 3 ${BENCH_ARGS:-} > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
if [ "${SKIP_NCU:-0}" != 1 ]; then
if [ "${SKIP_LAUNCHES:-0}" != 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python tools/profile_one.py 1e12 8 > $O/launches.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
  python bench.py --limit 1e11 --steps 1 --warmup 3 --no-cpu-baseline > $O/launches_bench.log 2>&1
fi
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_verify -s 1 -c 1 \
  -o $O/prof_verify -f python tools/profile_one.py 1e12 9 > $O/ncu_full.log 2>&1
fi
ls -la $O
