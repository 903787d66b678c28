"""Dev probe: alternate persistent and per-kernel steps in one TP layout, sync after each."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import admit, build_group, last_logits
from paper_2605_23945_b200.models import geometry

seq = [tuple(int(v) for v in x.split("x")) for x in sys.argv[1].split(",")]
tp = int(sys.argv[2]) if len(sys.argv) > 2 else 2
geom = geometry("mini-qwen")
ranks, runner = build_group(geom, tp, max_batch=96, num_slots=96, max_len=96, seed=4)
slots = [admit(ranks, i, [1 + i % 50, 2, 3], max_ctx=64) for i in range(80)]
for B, n in seq:
    bk = ranks[0].executor.bucket(B)
    runner.set_rows(bk, slots[:min(B, 80)])
    runner.step(bk, n)
    torch.cuda.synchronize()
    cm = ranks[0].executor.comm
    print(f"B={B} bucket={bk} persist={runner.persist_ok(bk)} ok: epoch={int(cm.epoch.item()) if cm else None} "
          f"ctr={cm.ctr.tolist() if cm else None} prog={ranks[0].executor.p_work[:24].view(torch.int64).tolist() if ranks[0].executor.p_work is not None else None}",
          flush=True)
