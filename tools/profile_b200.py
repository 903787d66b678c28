"""Run the B200 Offline Profiler for a model and write the reference-schema CSV table."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23945_b200.latency import save_table
from paper_2605_23945_b200.models import geometry
from paper_2605_23945_b200.profiler import profile_b200

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen2.5-7b")
ap.add_argument("--tps", default="1,2,4,8")
ap.add_argument("--token-cap", type=int, default=1 << 20)
ap.add_argument("--max-ctx", type=int, default=16384 + 128)
ap.add_argument("--budget", type=float, default=900.0)
ap.add_argument("--out", required=True)
a = ap.parse_args()
t0 = time.time()
tab = profile_b200(geometry(a.model), tuple(int(x) for x in a.tps.split(",")), a.token_cap, a.max_ctx, a.budget,
                   log=lambda m: print(f"[{time.time() - t0:7.1f}s] {m}", flush=True))
save_table(tab, a.out)
print(f"wrote {a.out}: {len(tab.points)} points in {time.time() - t0:.0f} s")
