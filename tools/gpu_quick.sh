cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python tools/quick_bench.py 1e12 > gpurun_out/qb.txt 2>&1
timeout 300 python tools/quick_bench.py 1e13 >> gpurun_out/qb.txt 2>&1
