"""CPU: the multi-GPU scaling model (tools/scaling_model.py) replays the
library's real per-rank tile lists; on one rank it reproduces the measured
single-GPU apply, and its row-band efficiencies stay within physical bounds."""

import os
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_scaling_model_cfg3():
    out = subprocess.run([sys.executable, "tools/scaling_model.py", "3", "1", "2"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    rows = {r["G"]: r for r in d["rows"]}
    assert 0.1 < rows[1]["apply_ms"] < 0.5          # measured: 0.20 ms on one B200
    assert 0 < rows[2]["efficiency"] <= 1.05
    assert len(rows[2]["per_rank_ms"]) == 2
