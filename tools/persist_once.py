"""Dev probe: a few graph-replayed persistent decode steps of one loopback rank (for ncu)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

name, tp, B, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
n = int(sys.argv[5]) if len(sys.argv) > 5 else 3
geom = geometry(name)
r, runner = loopback_rank(geom, tp, B, B, ctx + 256, B * ((ctx + 256) // 64 + 2))
slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(B)]
r.slots.pos[:] = ctx
bk = r.executor.bucket(B)
runner.set_rows(bk, slots)
runner.step(bk, 1)
runner.capture(bk)
runner.step(bk, n)
torch.cuda.synchronize()
print("done")
