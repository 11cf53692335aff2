cd "${GRAFT_REPO_ROOT:-/root/repo}"
: > gpurun_out/c5v.txt
for v in build/variants/*/; do n=$(basename $v); echo "== $n" >> gpurun_out/c5v.txt; GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=$v/libgoldbach_b200.so timeout 300 python tools/range_bench.py 4e18 1e11 2 2>&1 | grep "time=" | tail -1 | cut -c1-200 >> gpurun_out/c5v.txt; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_wheel.py -x -q -k "c5 or large or ceiling" > gpurun_out/pytest_c5.txt 2>&1; echo rc=$? >> gpurun_out/pytest_c5.txt
