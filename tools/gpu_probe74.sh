timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_a.json > /dev/null 2>&1
TPS_ATTN_EARLY=0 timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_b.json > /dev/null 2>&1
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_c.json > /dev/null 2>&1
python -c "
import json
for n in ('sb_a','sb_b','sb_c'):
    d=json.load(open('gpurun_out/'+n+'.json')); print(n, round(d['generation_time'],3), {k: round(v['ms_per_round'],3) for k,v in d['buckets'].items()})"
