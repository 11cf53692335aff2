# time every build/variants/* library on the C3 range (and LIMS)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
: > gpurun_out/variants.txt
for L in ${LIMS:-1e12}; do
for v in build/variants/*/; do
  n=$(basename $v)
  echo "== $n $L" >> gpurun_out/variants.txt
  GB_TOOLS_LIB_OVERRIDE=1 GB_LIB_PATH=$v/libgoldbach_b200.so timeout 300 python tools/quick_bench.py $L 2>&1 | grep "limit=" | tail -1 >> gpurun_out/variants.txt
done
done
