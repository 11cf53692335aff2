#!/usr/bin/env bash
# A/B of the bucket-sieve knobs at 1e12 / 1e13 (quick_bench, same checksums).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
for L in ${LIMITS:-1e13 1e12}; do
  for P in ${PBS:-0 131072 262144 524288 1048576}; do
    for F in 0; do
      echo "== L=$L GB_MASK_P=$P" >> $O/variants.txt
      GB_MASK_P=$P timeout 300 python tools/quick_bench.py $L 2>&1 | grep -v "^stats\|no stats" >> $O/variants.txt
    done
  done
done
