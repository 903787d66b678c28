"""Read a bench line (a driver BENCH_rNN.json, or a log whose last JSON line is bench.py's) and
decide the warp-shuffle GEMV's default: per tail bucket (`tail.per_batch`, TP8 loopback rank)
the default step vs the GEMV step, and the stage-level A/B (`gemv_stage` vs `value`).

python tools/gemv_decide.py BENCH_r02.json
"""
import json, sys


def load(path):
    text = open(path).read()
    try:
        d = json.loads(text)
        return d.get("parsed", d)
    except json.JSONDecodeError:
        lines = [l for l in text.splitlines() if l.startswith("{")]
        return json.loads(lines[-1])


line = load(sys.argv[1])
rows = []
for b, v in sorted((line.get("tail") or {}).get("per_batch", {}).items(), key=lambda kv: int(kv[0])):
    if "gemv_ms" in v:
        rows.append((int(b), v["ms"], v["gemv_ms"], v["ms"] / v["gemv_ms"]))
        print(f"TP8 B={b}: default {v['ms']:.3f} ms  gemv {v['gemv_ms']:.3f} ms  speed-up {v['ms'] / v['gemv_ms']:.3f}"
              f"  (HBM frac {v['frac']:.2f} -> {v['gemv_frac']:.2f})")
st = line.get("gemv_stage") or {}
if "value" in st:
    print(f"stage: default {line['value']:.3f} s  gemv {st['value']:.3f} s  speed-up {line['value'] / st['value']:.3f}")
wins = [b for b, _, _, s in rows if s > 1.02]
print("recommendation: GEMV_ROWS =", max(wins) if wins and (not st or st.get("value", 1e9) <= line["value"]) else 0)
