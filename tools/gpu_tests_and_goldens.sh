#!/usr/bin/env bash
# GPU test suite while the host cores generate reference goldens (the test
# suite needs the GPU, the golden generator only the CPU).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
if [ -n "$GOLD_PART" ]; then
  timeout ${GOLD_SECS:-1800} python oracle/make_big_goldens.py --set c4 --part $GOLD_PART --jobs ${GOLD_JOBS:-13} \
    --out $O/c4_${GOLD_PART/:/_}.tsv > $O/c4_gen_${GOLD_PART/:/_}.log 2>&1 &
  GP=$!
fi
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
if [ -n "$GOLD_PART" ]; then wait $GP; wc -l $O/c4_${GOLD_PART/:/_}.tsv; fi
