"""Dev probe: in-kernel timeline of one layer of the persistent decode step (loopback rank).

python tools/persist_trace.py <model> <tp> <B> <ctx> [layer]
Per event: min / median / max over CTAs of (mark - min(layer start)), microseconds.
"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import admit
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import loopback_rank

EV = ["layer start", "norm(in) ready", "QKV pieces done", "QKV ready", "attention done", "attention ready",
      "O pieces done", "norm slices done", "norm ready", "gate/up done", "act ready", "down done",
      "norm slices done", "step start", "step end", "-", "att: unit start", "att: q issued", "att: pages done",
      "att: partial out", "att: counted", "att: merged", "att: m/l loaded", "att: weights", "-", "-", "qkv: unit start", "qkv: mma done", "qkv: reduced",
      "qkv: epilogue done", "qkv: window loaded"]
name, tp, B, ctx = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
layer = int(sys.argv[5]) if len(sys.argv) > 5 else 1
geom = geometry(name)
r, runner = loopback_rank(geom, tp, B, B, ctx + 256, B * ((ctx + 256) // 64 + 2))
slots = [admit([r], i, [1, 2, 3], max_ctx=ctx + 200) for i in range(B)]
r.slots.pos[:] = ctx
bk = r.executor.bucket(B)
runner.set_rows(bk, slots)
ex = r.executor
ex.p_trace = torch.zeros((148, 32), dtype=torch.int64, device="cuda")
ex.p_trace_layer = layer
runner.step(bk, 1)
runner.capture(bk)
runner.step(bk, 5)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
runner.step(bk, 20)
ev1.record()
torch.cuda.synchronize()
print(f"{name} tp={tp} B={B} ctx={ctx}: step {ev0.elapsed_time(ev1) / 20 * 1e3:.1f} us (graph replay)")
t = ex.p_trace.cpu()
C = ex.p_ctas
t = t[:C].double()
m = t[:, 21] > 0
if m.any():
    i = int(torch.argmax(t[:, 21] * m))
    row = t[i]
    print("  last merging CTA", i, "G*100+Sa", int(row[25]),
          "us after counted:", [round(float(row[e] - row[20]) / 1e3, 2) for e in (22, 23, 21)])
q = t[:, 29] > 0
if q.any():
    i = int(torch.argmax(t[:, 29] * q))
    row = t[i]
    print("  slowest QKV CTA", i, "us after norm ready (event 1): start/window/mma/reduce/epilogue",
          [round(float(row[e] - row[1]) / 1e3, 2) for e in (26, 30, 27, 28, 29)],
          "producer issued QKV boxes first/last (us after norm ready):",
          round(float(row[31] - row[1]) / 1e3, 2), round(float(row[15] - row[1]) / 1e3, 2))
base = t[:, 0].min()
for e, nm in enumerate(EV):
    if nm == "-":
        continue
    col = t[:, e]
    if e > 15:
        ok = col > 0
        if not ok.any():
            continue
        col = col[ok]
    if e >= 13:
        b2 = t[:, 13].min()
        col = col - b2
        print(f"  {e:2d} {nm:20s} min {col.min() / 1e3:8.2f} med {col.median() / 1e3:8.2f} max {col.max() / 1e3:8.2f} (from step start)")
        continue
    col = col - base
    print(f"  {e:2d} {nm:20s} min {col.min() / 1e3:8.2f} med {col.median() / 1e3:8.2f} max {col.max() / 1e3:8.2f}")
