bash tools/gpu_quick.sh
LIMS="${LIMS:-1e12 1e13}" bash tools/gpu_variants.sh
if [ -n "$NCU" ]; then LIMS="1e12" bash tools/gpu_ncu.sh; fi
