bash tools/gpu_quick.sh
LIMS="1e12 1e13" bash tools/gpu_variants.sh
