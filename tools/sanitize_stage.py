"""compute-sanitizer target: one short adaptive stage in a virtual 4-rank world (TP1 -> 2 -> 4
live switches, LL allreduce, KV migration, graph replays), the tiny model.

compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_stage.py [graphs]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2605_23945_b200 import _native as nat
from paper_2605_23945_b200.cache_manager import World
from paper_2605_23945_b200.coordinator import GlobalCoordinator
from paper_2605_23945_b200.models import geometry
from test_gpu_coordinator import tiny_spec

graphs = len(sys.argv) > 1 and sys.argv[1] == "graphs"
geom = geometry("tiny")
spec = tiny_spec(geom, batch=8, l_max=24)
coord = GlobalCoordinator(spec, geom, World.virtual(4), seed=7, use_graphs=graphs)
rep, _ = coord.run()
nat.check_abort("sanitized stage")
sw = [(s["from_tp"], s["to_tp"]) for nr in rep.node_reports for s in nr["switches"]]
print(f"stage ok: {rep.tokens_generated} tokens, switches {sw}, graphs={graphs}")
