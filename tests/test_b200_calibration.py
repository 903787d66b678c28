"""presets/b200.cfg's Switch Executor constants follow from the committed config-5 sweep.

tools/calibrate_switch.py derives them from profiles/r2/switch_sweep_qwen7b.jsonl (the B200
sweep of the Switch Executor, 114 points); this pins the preset to that evidence so a later edit
of either cannot silently drift (Algorithm 1's switch term, tpshift/switchcost.py:76-139,
166-167, 234-242, reads these constants).
"""

import json
import os
import subprocess
import sys

from paper_2605_23945_b200.config import load_config

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_switch_constants_match_the_measured_sweep():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "calibrate_switch.py"),
                          os.path.join(ROOT, "profiles", "r2", "switch_sweep_qwen7b.jsonl")],
                         capture_output=True, text=True, check=True).stdout
    cal = json.loads(out)
    cfg = load_config("b200")
    assert cal["points"] >= 100
    # one-way pull rate: the NVLink peer copy x the copy engine's median efficiency, rounded to 2 digits
    assert abs(cfg.cluster.intra_bw_unidir - cal["intra_bw_unidir"]) <= 0.02 * cal["intra_bw_unidir"]
    # fixed control cost: the sweep's p90 of (switch device time - copy time), rounded up
    assert cal["t_fixed_control_ms"]["p90"] / 1e3 <= cfg.switch.t_fixed_control <= 1.5 * cal["t_fixed_control_ms"]["p90"] / 1e3
    # graph capture and communicator/layout build inside a switch: bounded by the measured maxima
    assert cfg.switch.graph.cost_per_bucket >= cal["graph_capture_in_switch_s"] / len(cfg.switch.graph.capture_buckets)
    assert cal["layout_build_in_switch_s"] <= cfg.switch.comm_init_cost <= 2 * cal["layout_build_in_switch_s"]
