timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_decode.py -x -q 2>&1 | tail -2
timeout 900 python tools/solo_step.py qwen2.5-7b 1 4,8,16,32,64 2048 "" 2>&1 | grep -v watchdog
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_early.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/sb_early.json')); print('stage', round(d['generation_time'],3), {k: round(v['ms_per_round'],3) for k,v in d['buckets'].items()})"
