#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out; mkdir -p $O
( for i in 1 2 3; do s=$(date +%s.%N); ./paper_2603_07850_b200/bin/goldbach --help > /dev/null; e=$(date +%s.%N); echo "help process $(echo "$e - $s" | bc) s"; done ) > $O/startup.txt 2>&1
( for i in 1 2; do s=$(date +%s.%N); python -c "import ctypes; ctypes.CDLL('paper_2603_07850_b200/libgoldbach_b200.so')"; e=$(date +%s.%N); echo "python+dlopen $(echo "$e - $s" | bc) s"; done ) >> $O/startup.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
  python tools/profile_one.py 4000000100000000000 9 > $O/launches_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_verify|k_large" -s 2 -c 2 \
  -o $O/prof_c5 -f python tools/profile_one.py 4000000100000000000 9 > $O/ncu_c5.log 2>&1
timeout ${GOLD_SECS:-1900} python oracle/make_big_goldens.py --set c4 --part 5000:10000 --jobs 16 --skip oracle/_ref/c4_done.tsv \
  --out $O/c4_part2.tsv > $O/c4_gen_part2.log 2>&1
wc -l $O/c4_part2.tsv
