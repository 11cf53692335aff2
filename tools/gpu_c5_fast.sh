#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
timeout 300 python tools/range_bench.py 4e18 1e11 3 2>&1 | grep -E "time=|kernel" | cut -c1-160 > $O/c5fast.txt
timeout 900 python -m pytest tests/test_gpu_bigranges.py tests/test_gpu_tile.py tests/test_gpu_parity.py tests/test_gpu_bucket.py -x -q > $O/pytest_c5fast.txt 2>&1; echo rc=$? >> $O/pytest_c5fast.txt
