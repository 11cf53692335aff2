#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in ${VARS:-m6_320k}; do
  for L in 1e12 1e13; do
    echo "== $V $L" >> $O/m6.txt
    GB_DEBUG_OPEN=1 GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/$V/libgoldbach_b200.so timeout 200 python tools/quick_bench.py $L 2>&1 | grep -E "time=|rror|cannot" | tail -2 | cut -c1-170 >> $O/m6.txt
  done
done

GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/m6_320k/libgoldbach_b200.so timeout 900 python -m pytest tests/test_gpu_tile.py tests/test_gpu_parity.py tests/test_gpu_wheel.py tests/test_gpu_random.py -x -q > $O/pytest_m6.txt 2>&1; echo rc=$? >> $O/pytest_m6.txt
