#!/usr/bin/env bash
# Round-2 closing call: strike variants, GPU suite (full C4/C5 records),
# 2-rank gloo bench on one GPU, bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in pred2 b563; do
  for L in 1e12 1e13; do
    echo "== $V $L" >> $O/final_var.txt
    GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/final_var.txt
  done
done
for L in 1e12 1e13; do echo "== default $L" >> $O/final_var.txt; timeout 300 python tools/quick_bench.py $L 2>&1 | grep -E "time=" | cut -c1-110 >> $O/final_var.txt; done
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
GB_BENCH_BACKEND=gloo GB_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --limit 1e11 --steps 2 --warmup 3 > $O/multirank_gloo.json 2> $O/multirank_gloo.err
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_1e12.json 2> $O/bench_1e12.err
timeout 900 python bench.py --limit 1e13 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_1e13.json 2> $O/bench_1e13.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
ls -la $O
