import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import admit, build_group
from paper_2605_23945_b200.models import geometry
PROMPTS = [[5, 17, 300, 9, 4000, 1, 2, 3], [42, 42, 42, 7, 7, 7, 1000, 2047]]
for name, tp, nsteps in [("tiny", 1, 20), ("tiny", 2, 20), ("mini-qwen", 1, 20), ("mini-qwen", 2, 20), ("tiny", 2, 80)]:
    geom = geometry(name)
    outs = []
    for graphs in (False, True):
        ranks, runner = build_group(geom, tp, max_batch=8, num_slots=4, max_len=128, seed=3, use_graphs=graphs)
        slots = [admit(ranks, i, p, max_ctx=len(p) + nsteps + 2) for i, p in enumerate(PROMPTS)]
        runner.set_rows(2, slots)
        runner.step(2, 1)
        if graphs:
            runner.capture(2)
        if len(sys.argv) > 1 and sys.argv[1] == "sync":
            for _ in range(nsteps):
                runner.step(2, 1)
                torch.cuda.synchronize()
        else:
            runner.step(2, nsteps)
        torch.cuda.synchronize()
        outs.append(ranks[0].slots.history[slots].cpu())
    d = (outs[0] != outs[1]).nonzero()
    print(name, tp, "equal" if d.numel() == 0 else f"first diff at {d[0].tolist()} of {d.shape[0]}", flush=True)
