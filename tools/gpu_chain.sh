#!/usr/bin/env bash
# First-index chain A/B on the C5 window; bounds probe (default, bounds
# variant, per-slot path); large-prime parity tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for V in "GB_LS_CHAIN=0" "GB_LS_CHAIN=1" "GB_LS_CHAIN=0" "GB_LS_CHAIN=1"; do
  echo "== $V" >> $O/chain_c5.txt
  env $V timeout 300 python tools/range_bench.py 4e18 1e11 3 2>&1 | grep -E "time=|kernel" | cut -c1-330 >> $O/chain_c5.txt
done
( echo "== default (row walk, first-index chain)"; timeout 500 python tools/ls_bounds_check.py
  echo "== bounds variant (GB_LS_BOUNDS + GB_STATS)"; GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=build/variants/bounds/libgoldbach_b200.so timeout 500 python tools/ls_bounds_check.py
  echo "== per-slot path (GB_LS_ROWS=0)"; GB_LS_ROWS=0 timeout 500 python tools/ls_bounds_check.py ) > $O/chain_bounds.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_bigranges.py tests/test_gpu_bucket.py tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_tile.py -x -q > $O/chain_pytest.txt 2>&1; echo "rc=$?" >> $O/chain_pytest.txt
