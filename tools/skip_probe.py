"""Dev probe: marginal in-graph cost of each launch kind (step time with that kind left out)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import build_group, admit
from paper_2605_23945_b200.models import geometry

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
batches = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 16, 64]
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
geom = geometry(name)
maxb = max(batches)
ranks, runner = build_group(geom, 1, max_batch=maxb, num_slots=maxb, max_len=ctx + 256, seed=0)
slots = [admit(ranks, i, [1, 2, 3], max_ctx=ctx + 200) for i in range(maxb)]
ex = ranks[0].executor
variants = [(), ("qkv_rope",), ("attention",), ("add_norm",), ("qkv_rope", "attention", "add_norm"), ("linear",)]
for B in batches:
    bk = ex.bucket(B)
    runner.set_rows(bk, slots[:B])
    base = None
    for skip in variants:
        ex.skip = frozenset(skip)
        runner.graphs.pop(bk, None)
        ranks[0].slots.pos[:] = ctx
        runner.step(bk, 1)
        runner.capture(bk)
        runner.step(bk, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record(); runner.step(bk, n); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        base = ms if base is None else base
        print(f"B={B:3d} ctx={ctx} skip={','.join(skip) or '-':35s} step {ms:.3f} ms  (delta {base - ms:+.3f})",
              flush=True)
    ex.skip = frozenset()
