for i in 1 2; do
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_def$i.json > /dev/null 2>&1
TPS_ATTN_MIN_BAL=1000 timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_split$i.json > /dev/null 2>&1
done
python -c "
import json
for n in ('sb_def1','sb_split1','sb_def2','sb_split2'):
    d=json.load(open('gpurun_out/'+n+'.json')); print(n, round(d['generation_time'],3), {k: round(v['ms_per_round'],3) for k,v in d['buckets'].items()})"
