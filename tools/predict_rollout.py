"""Predict the N-GPU generation stage on B200 from the measured Offline-Profiler table.

The reference's engine loop runs with TableBackend (measured B200 step/prefill times as
the ground truth) and the planner fitted to the same table: adaptive (Algorithm 1) vs
every fixed TP. Writes one JSON line per N.
"""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2605_23945_b200.engine import TableBackend, run
from paper_2605_23945_b200.latency import load_table

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen2.5-7b")
ap.add_argument("--table", default="", help="profile CSV (default presets/b200_<model>_profile.csv)")
ap.add_argument("--initial-tp", type=int, default=1)
ap.add_argument("--gpus", default="1,2,4,8")
ap.add_argument("--per-gpu-batch", type=int, default=64)
ap.add_argument("--l-max", type=int, default=8192)
ap.add_argument("--tp-list", default="", help="Algorithm 1 candidates (default 1,N as bench.py)")
ap.add_argument("--raw", action="store_true", help="the measured table as is (default: monotone fit, as bench.py)")
a = ap.parse_args()
tab = load_table(a.table or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "paper_2605_23945_b200", "presets", f"b200_{a.model}_profile.csv"))
if not a.raw:
    from paper_2605_23945_b200.profiler import monotone_table
    tab = monotone_table(tab)
for n in (int(x) for x in a.gpus.split(",")):
    if n % a.initial_tp:
        continue
    ns = argparse.Namespace(model=a.model, per_gpu_batch=a.per_gpu_batch, l_max=a.l_max, prompt_len=512, seed=4,
                            tp_list=a.tp_list, initial_tp=a.initial_tp)
    spec, geom = bench.build_spec(ns, n)
    rep = run(spec, tab, TableBackend(spec, tab))
    out = {"model": a.model, "table": "raw" if a.raw else "monotone", "gpus": n, "per_gpu_batch": a.per_gpu_batch, "l_max": a.l_max, "tp_list": list(spec.controller.tp_list), "adaptive_s": round(rep.generation_time, 3),
           "switches": [[s["from_tp"], s["to_tp"], s["round"], round(s["breakdown"]["total"], 3)]
                        for nr in rep.node_reports for s in nr["switches"]], "static_s": {}}
    for tp in (1, 2, 4, 8):
        if n % tp == 0 and tp >= a.initial_tp:
            s2 = dataclasses.replace(spec, mode="static", initial_tp=tp)
            out["static_s"][tp] = round(run(s2, tab, TableBackend(s2, tab)).generation_time, 3)
    print(json.dumps(out), flush=True)
