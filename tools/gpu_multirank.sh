# Multi-rank path check on a 1-GPU box: 2 ranks share GPU 0 over gloo
# (shared work-stealing cursor, all-gather merge, max-over-ranks timing).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
GB_BENCH_BACKEND=gloo GB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 \
  --limit 1e11 > gpurun_out/multirank.json 2> gpurun_out/multirank.err
echo "rc=$?" >> gpurun_out/multirank.err
python bench.py --gpus 1 --steps 2 --warmup 3 --limit 1e11 --no-cpu-baseline > gpurun_out/single_1e11.json 2>> gpurun_out/multirank.err
