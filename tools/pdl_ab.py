"""Dev probe: decode-step time with programmatic dependent launch on vs off."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.group import build_group, admit
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import step_probe, gemm_probe

geom = geometry(sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b")
ctx = 2048
ranks, runner = build_group(geom, 1, max_batch=64, num_slots=64, max_len=ctx + 256, seed=0)
slots = [admit(ranks, i, [1, 2, 3], max_ctx=ctx + 200) for i in range(64)]
ex = ranks[0].executor
for pdl in (1, 0, 1):
    nat.lib().tps_set_pdl(pdl)
    runner.graphs.clear()
    for B in (1, 16, 64):
        ranks[0].slots.pos[:] = ctx
        bk = ex.bucket(B)
        runner.set_rows(bk, slots[:B])
        ms = step_probe(runner, bk, 30)
        print(f"pdl={pdl} B={B} step {ms:.3f} ms", flush=True)
for B in (1, 16, 64):
    g = gemm_probe(ex, B)
    print(B, {k: round(v['bytes'] / v['ms'] / 1e6) for k, v in g.items() if k != 'total'}, round(g['total']['gbps']))
