"""CPU: bench.py's reference arm (the reference CPU path timed on this
host) prints the contract's JSON line; the frozen roofline formula."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_alg_bytes_formula_frozen_points():
    # B = 24.7 (1e8), 26.6 (1e10), 28.3 (1e12), 29.2 (1e13), 34.4 (4e18)
    for n, b in [(1e8, 24.7), (1e10, 26.6), (1e12, 28.3), (1e13, 29.2), (4e18, 34.4)]:
        assert abs(bench.alg_bytes_per_even(n) - b) < 1e-9
    assert 26.6 < bench.alg_bytes_per_even(1e11) < 28.3


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "goldbach_ref")),
                    reason="oracle/_ref not built")
def test_reference_arm_line():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--limit", "1e9", "--seg-size", "20000000", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-1000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True
