"""Where a cold `bin/goldbach LIMIT --gpus=K --json` process spends its wall
time: spawn -> each GB_DEBUG_OPEN timing line (stderr, timestamped on
arrival) -> exit.

    python tools/cli_timing.py [limit] [gpus] [reps]
"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2603_07850_b200", "bin", "goldbach")
limit = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**12
gpus = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
env = dict(os.environ, GB_DEBUG_OPEN="1")
for _ in range(reps):
    t0 = time.perf_counter()
    p = subprocess.Popen([EXE, str(limit), f"--gpus={gpus}", "--json"], stdout=subprocess.PIPE,
                         stderr=subprocess.PIPE, text=True, env=env)
    for line in p.stderr:
        print(f"  +{time.perf_counter() - t0:7.3f} s  {line.rstrip()}", flush=True)
    out = p.stdout.read()
    rc = p.wait()
    print(f"exit rc={rc} after {time.perf_counter() - t0:.3f} s; json: {out.strip()[:160]}", flush=True)
