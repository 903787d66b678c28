"""bench.py --impl reference (the CPU arm the driver runs beside ours) prints one JSON line with
the contract's keys, on the CPU (no GPU needed): the CPU oracle's full-depth steps composed over
the stage, the decision layer through the restated and the unmodified reference, and the CPU
switch baseline."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert cb["switch"]["gbps"] > 0
    dl = cb["decision_layer"]
    assert dl["evaluate_ms"] > 0
    if "unavailable" not in dl["reference_impl"]:
        assert dl["reference_impl"]["report_identical"] and dl["reference_impl"]["decision_identical"]
