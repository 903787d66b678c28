"""How much the N-GPU predictions depend on the modeled NVLink hop (DESIGN 5.3).

The TP>1 rows of the Offline Profiler's tables are loopback-rank step times plus
`profiler.nvlink_adjust` (per allreduce: one hop latency + the pushed bytes at the peer-copy
bandwidth; 1.5 us and 770 GB/s when profiled). This re-prices every TP>1 decode point with
other (hop, bandwidth) pairs and re-runs the stage predictions (adaptive vs every fixed TP).

python tools/nvlink_sensitivity.py > profiles/r2/nvlink_sensitivity.jsonl
"""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2605_23945_b200 import profiler as P
from paper_2605_23945_b200.engine import TableBackend, run
from paper_2605_23945_b200.latency import ProfilePoint, load_table, table_from_points
from paper_2605_23945_b200.models import geometry

CONFIGS = [("qwen2.5-7b", 64, 8192, 1, "1,8"), ("llama3-8b", 32, 16384, 1, "1,2,4,8"),
           ("qwen2.5-32b", 16, 16384, 2, "2,4,8")]
SETTINGS = [(1.5e-6, 770.0), (3e-6, 770.0), (6e-6, 770.0), (1.5e-6, 450.0), (6e-6, 450.0)]


def repriced(tab, geom, hop, gbps):
    base = (P.NVLINK_HOP_S, P.NVLINK_GBPS)
    pts = []
    for p in tab.points:
        d = p.decode_latency
        if p.tp > 1:
            P.NVLINK_HOP_S, P.NVLINK_GBPS = base
            d -= P.nvlink_adjust(geom, p.tp, p.batch)
            P.NVLINK_HOP_S, P.NVLINK_GBPS = hop, gbps
            d += P.nvlink_adjust(geom, p.tp, p.batch)
        pts.append(ProfilePoint(p.tp, p.batch, p.ctx_len, d, p.prefill_latency))
    P.NVLINK_HOP_S, P.NVLINK_GBPS = base
    return table_from_points(pts, tab.token_cap)


here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for model, pgb, l_max, t0, tps in CONFIGS:
    geom = geometry(model)
    raw = load_table(os.path.join(here, "paper_2605_23945_b200", "presets", f"b200_{model}_profile.csv"))
    for hop, gbps in SETTINGS:
        tab = P.monotone_table(repriced(raw, geom, hop, gbps))
        ns = argparse.Namespace(model=model, per_gpu_batch=pgb, l_max=l_max, prompt_len=512, seed=4, tp_list=tps,
                                initial_tp=t0)
        spec, _ = bench.build_spec(ns, 8)
        rep = run(spec, tab, TableBackend(spec, tab))
        static = {}
        for tp in (1, 2, 4, 8):
            if tp >= t0:
                s2 = dataclasses.replace(spec, mode="static", initial_tp=tp)
                static[tp] = round(run(s2, tab, TableBackend(s2, tab)).generation_time, 3)
        best = min(static, key=static.get)
        print(json.dumps({"model": model, "gpus": 8, "tp_list": tps, "hop_us": hop * 1e6, "nvlink_gbps": gbps,
                          "adaptive_s": round(rep.generation_time, 3), "best_fixed_tp": best,
                          "best_fixed_s": static[best], "static_s": static,
                          "switches": sum(len(nr["switches"]) for nr in rep.node_reports)}), flush=True)
