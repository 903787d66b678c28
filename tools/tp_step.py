"""Dev probe: virtual TP group (all ranks on one GPU) step time, fused vs unfused allreduce epilogue."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import build_group, admit
from paper_2605_23945_b200.models import geometry

name = sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b"
tp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
batches = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 16, 64]
ctx = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
geom = geometry(name)
maxb = max(batches)
ranks, runner = build_group(geom, tp, max_batch=maxb, num_slots=maxb, max_len=ctx + 256, seed=0)
slots = [admit(ranks, i, [1, 2, 3], max_ctx=ctx + 200) for i in range(maxb)]
for B in batches:
    bk = ranks[0].executor.bucket(B)
    runner.set_rows(bk, slots[:B])
    for skip in ((), ("fuse_push",)):
        for r in ranks:
            r.executor.skip = frozenset(skip)
            r.slots.pos[:] = ctx
        runner.graphs.pop(bk, None)
        runner.step(bk, 1)
        runner.capture(bk)
        runner.step(bk, 3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record(); runner.step(bk, n); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{name} tp={tp} B={B:3d} ctx={ctx} {'unfused' if skip else 'fused  '} step {ms:.3f} ms "
              f"({ms / tp:.3f} ms per rank-share) kernels/step {runner.kernels_per_step(bk)}", flush=True)
