"""Dev probe: where a bench stage's time goes (prefill, decode per active-batch bucket) vs the HBM floor.

python tools/stage_breakdown.py [--model qwen2.5-7b] [--per-gpu-batch 64] [--l-max 8192]
Prints per bucket: rounds, mean ms/round, algorithmic bytes/round (weights + KV read), GB/s, frac of peak.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2605_23945_b200.cache_manager import World  # noqa: E402
from paper_2605_23945_b200.coordinator import GlobalCoordinator  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-7b")
    ap.add_argument("--per-gpu-batch", type=int, default=64)
    ap.add_argument("--l-max", type=int, default=8192)
    ap.add_argument("--prompt-len", type=int, default=512)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    spec, geom = bench.build_spec(a, a.gpus)
    coord = GlobalCoordinator(spec, geom, World.virtual(a.gpus), seed=0)
    coord.run()
    rep, meas = coord.run()
    ex = next(iter(coord.backend.ranks.values())).executor
    wbytes = ex.w.nbytes - geom.vocab * geom.hidden * 2  # embedding rows are gathered
    peak, _ = bench.peaks()
    nr = rep.node_reports[0]
    # reconstruct per-round active batch and context sums from the engine's event log
    grp = meas["groups"]
    out = {"generation_time": rep.generation_time, "prefill_s": None, "buckets": {}}
    for key, g in grp.items():
        out["prefill_s"] = g["prefill"]
        rounds = np.array(g["rounds"])
        dt = np.diff(np.concatenate([[g["prefill"]], rounds]))
        # active batch per round from step-block events
        act = []
        for ev in nr["events"]:
            if ev["type"] == "step-block":
                lo, hi = (int(x) for x in ev["detail"].split("=")[1].split(".."))
                act += [ev["active"]] * (hi - lo)
        act = np.array(act[:len(dt)])
        for B in sorted(set(act.tolist())):
            m = act == B
            bk = ex.bucket(B)
            d = out["buckets"].setdefault(bk, {"rounds": 0, "s": 0.0})
            d["rounds"] += int(m.sum())
            d["s"] += float(dt[m].sum())
    for bk, d in out["buckets"].items():
        d["ms_per_round"] = d["s"] / d["rounds"] * 1e3
        d["weights_gbps"] = wbytes / (d["ms_per_round"] / 1e3) / 1e9
    out["decode_s"] = sum(d["s"] for d in out["buckets"].values())
    out["weights_GB"] = wbytes / 1e9
    out["weights_floor_s"] = sum(d["rounds"] for d in out["buckets"].values()) * wbytes / (peak * 1e6) / 1e3
    print(json.dumps(out, indent=1))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
