"""Dev probe: projection GEMM GB/s per family and batch (bench.py's roofline probe, itemised)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_23945_b200.group import build_group
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import gemm_probe
geom = geometry(sys.argv[1] if len(sys.argv) > 1 else "qwen2.5-7b")
ranks, runner = build_group(geom, 1, max_batch=64, num_slots=64, max_len=512, seed=0)
ex = ranks[0].executor
for B in (1, 16, 32, 64):
    g = gemm_probe(ex, B, reps=3)
    print(B, {k: (round(v["bytes"] / v["ms"] / 1e6), v.get("splits")) for k, v in g.items() if k != "total"},
          "total", round(g["total"]["gbps"]), flush=True)
