#!/usr/bin/env bash
# Builds the UNMODIFIED reference (compiled from its sources where they lie
# under /root/reference/proj -- nothing is copied) into oracle/_ref/:
#   goldbach_ref  the reference CLI (proj/tools/main.cpp), used as the CPU
#                 baseline arm of bench.py (--impl reference, cpu_baseline)
#   libref.so     reference library + oracle/ref_shim.cpp (golden generator)
# Flags are the reference's CMake Release flags (proj/CMakeLists.txt:12 plus
# -O3 -DNDEBUG).  The only header the reference tree lacks is nlohmann json
# (proj/CMakeLists.txt:5 expects vendor/); the copy bundled with
# cudnn_frontend in this image (v3.11.3) is used.  TEST INFRASTRUCTURE ONLY.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
R="${GB_REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$R/src" ]; then
  echo "build_ref: reference sources not present at $R; skipping" >&2
  exit 0
fi
J=""
for cand in \
  /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann \
  $(python3 -c 'import site,sys;print(" ".join(p+"/include/cudnn_frontend/thirdparty/nlohmann" for p in site.getsitepackages()))' 2>/dev/null); do
  if [ -f "$cand/json.hpp" ]; then J="$cand"; break; fi
done
if [ -z "$J" ]; then echo "build_ref: json.hpp not found" >&2; exit 1; fi
mkdir -p "$OUT"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O3 -DNDEBUG -Wall -Wextra -pthread"
LIB_SRCS="$R/src/oddbits.cpp $R/src/primality.cpp $R/src/sieve.cpp $R/src/verifier.cpp $R/src/pool.cpp"
if [ ! -x "$OUT/goldbach_ref" ] || [ "$0" -nt "$OUT/goldbach_ref" ]; then
  $CXX $FLAGS -I"$R/include" -I"$J" $R/src/*.cpp "$R/tools/main.cpp" -o "$OUT/goldbach_ref"
fi
if [ ! -f "$OUT/libref.so" ] || [ "$HERE/ref_shim.cpp" -nt "$OUT/libref.so" ]; then
  $CXX $FLAGS -fPIC -shared -I"$R/include" "$HERE/ref_shim.cpp" $LIB_SRCS -o "$OUT/libref.so"
fi
echo "build_ref: ok ($OUT)"
