timeout 900 python -m pytest tests/test_gpu_coordinator.py tests/test_gpu_decode.py -x -q 2>&1 | tail -1
for o in sample position; do timeout 600 python tools/stage_breakdown.py --prefill-order $o --out gpurun_out/sb_$o.json > /dev/null 2>&1; done
python -c "
import json
for n in ('sb_sample','sb_position'):
    d=json.load(open('gpurun_out/'+n+'.json')); print(n, 'stage', round(d['generation_time'],3), 'prefill', round(d['prefill_s'],3))"
