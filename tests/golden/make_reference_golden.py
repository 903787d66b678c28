"""Generate tests/golden/reference_decisions.json from the reference implementation itself.

Imports the read-only reference package `tpshift` (/root/reference/pkg/src) --
only possible in the build container -- and records, for fixed seeded inputs:
  * whole-stage SimReport / ComparisonReport JSON (sha256 + key scalars) for
    several scenarios and modes (the Global Coordinator loop),
  * Algorithm 1 decisions (evaluate) on random node states,
  * assign_merged_groups placements, compute_merged_bs, est_rem_time values,
  * switch-cost quotes, reshard-plan volumes, profile-table CSV digests,
  * sample_response_lengths streams.
Floats are stored with repr() so the parity tests compare bit-exactly.

    python tests/golden/make_reference_golden.py
"""

import hashlib
import io
import json
import os
import random
import sys
import tempfile
from dataclasses import replace

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
import tpshift as T  # noqa: E402


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def f(x):
    return repr(float(x))


def scenario_cases():
    a40 = T.load_config("paper_a40")
    h100 = T.load_config("paper_h100")
    out = []
    base = T.build_scenario(a40)
    out.append(("a40-default", "paper_a40", {}))
    out.append(("a40-lmax8k-seed1", "paper_a40", {"l_max": 8192, "seed": 1}))
    out.append(("a40-static-tp2", "paper_a40", {"mode": "static"}))
    out.append(("a40-naive", "paper_a40", {"mode": "naive-switch", "l_max": 12288}))
    out.append(("a40-b32-tp1", "paper_a40", {"global_batch": 32, "initial_tp": 1, "seed": 9, "l_max": 4096}))
    out.append(("h100-default", "paper_h100", {}))
    out.append(("h100-b384-8k-tp1", "paper_h100", {"global_batch": 384, "l_max": 8192, "initial_tp": 1}))
    del base
    return out, {"paper_a40": a40, "paper_h100": h100}


def main():
    gold = {"scenarios": {}, "compare": {}, "evaluate": [], "assign": [], "est_rem": [], "quotes": [],
            "plans": [], "lengths": [], "tables": {}}
    cases, cfgs = scenario_cases()
    tables = {}
    for name, cfg in cfgs.items():
        spec = T.build_scenario(cfg)
        tables[name] = T.build_profile(spec)
        buf = tempfile.NamedTemporaryFile(suffix=".csv", delete=False)
        buf.close()
        T.save_table(tables[name], buf.name)
        gold["tables"][name] = sha(open(buf.name).read())
        os.unlink(buf.name)
    for name, preset, ov in cases:
        spec = T.build_scenario(cfgs[preset], **ov)
        rep = T.run(spec, tables[preset])
        js = rep.to_json()
        gold["scenarios"][name] = {"preset": preset, "overrides": ov, "sha256": sha(js),
                                   "generation_time": f(rep.generation_time), "eval_count": rep.eval_count,
                                   "tokens": rep.tokens_generated,
                                   "switches": [(s["from_tp"], s["to_tp"], s["round"])
                                                for nr in rep.node_reports for s in nr["switches"]]}
    for name, preset, ov in (("a40-compare", "paper_a40", {}), ("h100-compare-12k", "paper_h100", {"l_max": 12288})):
        spec = T.build_scenario(cfgs[preset], **ov)
        # (the reference naive-switch mode trips its own pool assertion when the
        # target layout is cold, so compare() is recorded without include_naive)
        cr = T.compare(spec, tables[preset])
        gold["compare"][name] = {"preset": preset, "overrides": ov,
                                 "sha256": sha(json.dumps(cr.to_json_dict(), sort_keys=True)),
                                 "speedup": f(cr.speedup), "best_static_tp": cr.best_static_tp}

    # random node states for Algorithm 1 / merge-and-redistribute
    rng = random.Random(2026)
    a40 = cfgs["paper_a40"]
    pred = T.fit_predictor(tables["paper_a40"])
    for case in range(160):
        tp = rng.choice([1, 2, 4, 8])
        dp = 8 // tp
        samples = []
        sid = 0
        for g in range(dp):
            for _ in range(rng.randint(0, 12)):
                ctx = rng.randint(16, 14000)
                samples.append((sid, g, ctx))
                sid += 1
        if not samples:
            samples.append((0, 0, 700))
        statuses = []
        for g in range(dp):
            mem = tuple(T.Sample(id=i, prompt_len=c, target_response_len=1, intra_dp_group=gg)
                        for i, gg, c in samples if gg == g)
            statuses.append(T.BatchStatus(node_id=0, group_index=g, samples=mem))
        l_gen = rng.randint(0, 15000)
        warm = [(tp, dp)] + ([(8, 1)] if rng.random() < 0.5 else [])
        pool = T.CommGroupPool.fresh(a40.switch.comm_init_cost, warm=tuple(warm))
        use_oracle = case % 4 == 3
        p = T.OracleLatencyModel(T.build_hardware_model(T.build_scenario(a40))) if use_oracle else pred
        params = replace(a40.controller, chunk_steps=rng.choice([1, 7, 64]))
        dec = T.evaluate(params, p, pool, a40.switch, statuses, T.ParallelConfig.for_cluster(a40.cluster, tp),
                         16384, l_gen, a40.model, a40.cluster, naive_mode=(case % 11 == 5))
        gold["evaluate"].append({
            "samples": samples, "tp": tp, "l_gen": l_gen, "warm": warm, "oracle": use_oracle,
            "chunk": params.chunk_steps, "naive": case % 11 == 5, "action": dec.action,
            "target": dec.target.tp if dec.target else None, "t_cur": f(dec.t_cur), "t_best": f(dec.t_best),
            "evaluated": [(c.tp, f(c.t_rem), f(c.t_switch), f(c.t_total)) for c in dec.evaluated],
            "breakdown": ({k: (f(v) if isinstance(v, float) else v) for k, v in dec.breakdown.as_dict().items()}
                          if dec.breakdown else None)})
        for tgt in (1, 2, 4, 8):
            merged = T.assign_merged_groups(statuses, tgt, a40.cluster)
            gold["assign"].append({"case": case, "tgt": tgt, "groups": [[s.id for s in m] for m in merged]})
        rbs = [st.active_count for st in statuses]
        gold["assign"][-1]["merged_bs"] = {str(t): T.compute_merged_bs(rbs, t, a40.cluster) for t in (1, 2, 4, 8)}
        if l_gen < 16384:
            gold["est_rem"].append({"case": case, "val": f(T.est_rem_time(pred, tp, statuses, 16384, l_gen, 64))})

    # switch-cost quotes and plan volumes
    for tp_src in (1, 2, 4, 8):
        for tp_tgt in (1, 2, 4, 8):
            if tp_src == tp_tgt:
                continue
            for n, ctx in ((9, 12288), (1, 600), (40, 3000)):
                probe = [T.Sample(id=i, prompt_len=512, target_response_len=ctx - 512, generated_len=ctx - 512)
                         for i in range(n)]
                pool = T.CommGroupPool.fresh(0.3, warm=((tp_tgt, 8 // tp_tgt),) if n % 2 else ())
                q = T.total_switch_cost(pred, pool, a40.switch, probe, tp_src, tp_tgt, a40.model, a40.cluster)
                gold["quotes"].append({"src": tp_src, "tgt": tp_tgt, "n": n, "ctx": ctx,
                                       "q": {k: (f(v) if isinstance(v, float) else v)
                                             for k, v in q.as_dict().items()}})
            wp = T.plan_weight_reshard(a40.model, T.ShardLayout(tp_src, 4096), T.ShardLayout(tp_tgt, 4096))
            ks = [T.Sample(id=i, prompt_len=512, target_response_len=99, generated_len=100 * i,
                           intra_dp_group=i % (8 // tp_src)) for i in range(7)]
            kp = T.plan_kv_migration(ks, a40.model, tp_src, 8 // tp_src, tp_tgt)
            gold["plans"].append({"src": tp_src, "tgt": tp_tgt, "w_total": wp.total_per_rank_bytes,
                                  "w_peak": wp.peak_working_bytes, "kv_total": kp.total_per_rank_bytes,
                                  "kv_peak": kp.peak_working_bytes, "w_describe": sha(wp.describe())})
    for seed in (0, 4, 123):
        for dist in ("default", "scaled8k", "lognormal", "cdf"):
            if dist == "default":
                d = T.LengthDistribution.default()
            elif dist == "scaled8k":
                sh = np.log(24576 / 8192)
                d = T.LengthDistribution.mixture(8.847867 - sh, 0.12, 9.852194 - sh, 0.10, 0.023422, 8192)
            elif dist == "lognormal":
                d = T.LengthDistribution.lognormal(7.0, 0.8, 16384)
            else:
                d = T.LengthDistribution.empirical([(100, 0.2), (1000, 0.7), (5000, 1.0)], 5000)
            gold["lengths"].append({"seed": seed, "dist": dist,
                                    "sha256": sha(json.dumps(T.sample_response_lengths(d, 1000, seed)))})
    with open(os.path.join(HERE, "reference_decisions.json"), "w") as fh:
        json.dump(gold, fh, sort_keys=True, separators=(",", ":"))
    print("wrote reference_decisions.json",
          {k: len(v) for k, v in gold.items()})


if __name__ == "__main__":
    main()
