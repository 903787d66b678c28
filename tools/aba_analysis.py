"""What Algorithm 1's A -> B -> A switch pairs are worth (analysis only; the product keeps the
reference's rule). The same predicted stage (reference loop over the measured table, switches
realised at the Switch Executor's measured rates) is run twice: as is, and with every decision
that would return to the previous degree within `--window` rounds of the last switch vetoed
("stay"). Prints both stage times and switch counts.

python tools/aba_analysis.py --model llama3-8b --per-gpu-batch 32 --l-max 16384 --tp-list 1,2,4,8
"""
import argparse, dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2605_23945_b200 import engine as E
from paper_2605_23945_b200.controller import SwitchDecision
from paper_2605_23945_b200.engine import TableBackend, run
from paper_2605_23945_b200.latency import load_table
from paper_2605_23945_b200.profiler import monotone_table

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="llama3-8b")
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--per-gpu-batch", type=int, default=32)
ap.add_argument("--l-max", type=int, default=16384)
ap.add_argument("--tp-list", default="1,2,4,8")
ap.add_argument("--initial-tp", type=int, default=1)
ap.add_argument("--window", type=int, default=1000)
a = ap.parse_args()
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tab = monotone_table(load_table(os.path.join(here, "paper_2605_23945_b200", "presets", f"b200_{a.model}_profile.csv")))
ns = argparse.Namespace(model=a.model, per_gpu_batch=a.per_gpu_batch, l_max=a.l_max, prompt_len=512, seed=4,
                        tp_list=a.tp_list, initial_tp=a.initial_tp)
spec, _ = bench.build_spec(ns, a.gpus)


def stage(veto: bool):
    real = E.evaluate
    hist = {"prev": None, "last_round": -10 ** 9, "tp": spec.initial_tp}

    def vetoing(params, pred, pool, calib, statuses, current, l_max, l_gen, *rest, **kw):
        d = real(params, pred, pool, calib, statuses, current, l_max, l_gen, *rest, **kw)
        if d.action == "switch":
            if veto and d.target.tp == hist["prev"] and l_gen - hist["last_round"] < a.window:
                return SwitchDecision("stay", None, d.t_cur, d.t_cur, None, d.evaluated)
            hist["prev"], hist["last_round"] = current.tp, l_gen
        return d
    E.evaluate = vetoing
    try:
        rep = run(spec, tab, TableBackend(spec, tab))
    finally:
        E.evaluate = real
    sw = [(s["from_tp"], s["to_tp"], s["round"]) for nr in rep.node_reports for s in nr["switches"]]
    return rep.generation_time, sw


t0, sw0 = stage(False)
t1, sw1 = stage(True)
print(json.dumps({"model": a.model, "gpus": a.gpus, "tp_list": a.tp_list, "window_rounds": a.window,
                  "reference_rule_s": round(t0, 3), "switches": len(sw0),
                  "aba_vetoed_s": round(t1, 3), "switches_vetoed": len(sw1), "vetoed_sequence": sw1}))
