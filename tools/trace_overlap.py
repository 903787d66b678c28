"""Dev probe: do consecutive CUDA-graph replays of the decode step overlap (PDL across graph launches)?"""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank
name, tp, B, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
geom = geometry(name)
r, runner = loopback_rank(geom, tp, B, B, ctx + 256, B * ((ctx + 256) // 64 + 2))
slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(B)]
r.slots.pos[:] = ctx
bk = r.executor.bucket(B)
runner.set_rows(bk, slots)
runner.step(bk, 1); runner.capture(bk); runner.step(bk, 3); torch.cuda.synchronize()
cap = 4096
rec = torch.zeros(cap * 4, dtype=torch.int64, device="cuda")
ctr = torch.zeros(1, dtype=torch.int32, device="cuda")
nat.check(nat.lib().tps_trace_enable(rec.data_ptr(), ctr.data_ptr(), cap))
runner.step(bk, 2)
torch.cuda.synchronize()
nat.check(nat.lib().tps_trace_enable(None, None, 0))
n = int(ctr.item())
R = rec[:4 * n].view(n, 4).cpu().tolist()
k = n // 2
last1 = R[k - 1]
first2 = R[k]
print(f"{n} records; replay 1 last kernel kind {last1[0]} exit {last1[3]}; replay 2 first kernel kind {first2[0]} "
      f"entry {first2[1]} -> gap {(first2[1] - last1[3]) / 1e3:.2f} us (negative = overlap)")
mx = max(x[3] for x in R[:k])
early = [x for x in R[k:] if x[1] < mx]
print(f"replay-2 launches entering before replay 1 finished: {len(early)}")
