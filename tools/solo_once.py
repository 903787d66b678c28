"""One solo TP-k rank: eager step, capture, N graph replays (for ncu launch lists)."""
import sys, torch
sys.path.insert(0, ".")
from tools.solo_step import solo
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry
name, tp, B, ctx, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
geom = geometry(name)
r, runner = solo(geom, tp, B, ctx)
slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(B)]
r.slots.pos[:] = ctx
bk = r.executor.bucket(B)
runner.set_rows(bk, slots)
runner.step(bk, 1)
runner.capture(bk)
runner.step(bk, reps)
torch.cuda.synchronize()
print("kernels/step", runner.kernels_per_step(bk))
