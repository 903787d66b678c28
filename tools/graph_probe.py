"""Dev probe: graph-replayed decode vs eager decode, token histories compared.

python tools/graph_probe.py [sync]   -- small batches (cluster attention form)
python tools/graph_probe.py wide     -- B = 16 / 40 / 64 (split and page-balanced forms)
"""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import admit, build_group
from paper_2605_23945_b200.models import geometry

mode = sys.argv[1] if len(sys.argv) > 1 else ""
if mode == "wide":
    g = torch.Generator().manual_seed(0)
    cases = [("mini-qwen", tp, B, 24) for tp in (1, 2) for B in (16, 40, 64)]
else:
    cases = [("tiny", 1, 2, 20), ("tiny", 2, 2, 20), ("mini-qwen", 1, 2, 20), ("mini-qwen", 2, 2, 20), ("tiny", 2, 2, 80)]
for name, tp, B, nsteps in cases:
    geom = geometry(name)
    if mode == "wide":
        prompts = torch.randint(0, geom.vocab, (B, 8), generator=g).tolist()
    else:
        prompts = [[5, 17, 300, 9, 4000, 1, 2, 3], [42, 42, 42, 7, 7, 7, 1000, 2047]]
    outs = []
    for graphs in (False, True):
        ranks, runner = build_group(geom, tp, max_batch=64, num_slots=B + 2, max_len=128, seed=3, use_graphs=graphs)
        slots = [admit(ranks, i, p, max_ctx=len(p) + nsteps + 2) for i, p in enumerate(prompts)]
        bk = ranks[0].executor.bucket(B)
        runner.set_rows(bk, slots)
        runner.step(bk, 1)
        if graphs:
            runner.capture(bk)
        if mode == "sync":
            for _ in range(nsteps):
                runner.step(bk, 1)
                torch.cuda.synchronize()
        else:
            runner.step(bk, nsteps)
        torch.cuda.synchronize()
        outs.append(ranks[0].slots.history[slots].cpu())
    d = (outs[0] != outs[1]).nonzero()
    print(name, "tp", tp, "B", B, "equal" if d.numel() == 0 else f"first diff at {d[0].tolist()} of {d.shape[0]}",
          flush=True)
