for ctx in 768 2048; do timeout 900 python tools/solo_step.py qwen2.5-7b 1 16,32,48,64 $ctx "" 2>&1 | grep -v watchdog | sed 's/^/st3 /'; done
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_st3.json > /dev/null 2>&1
cp paper_2605_23945_b200/libtpshift_b200.so /tmp/st3.so; cp tools/lib_st2.so paper_2605_23945_b200/libtpshift_b200.so
for ctx in 768 2048; do timeout 900 python tools/solo_step.py qwen2.5-7b 1 16,32,48,64 $ctx "" 2>&1 | grep -v watchdog | sed 's/^/st2 /'; done
timeout 600 python tools/stage_breakdown.py --out gpurun_out/sb_st2.json > /dev/null 2>&1
cp /tmp/st3.so paper_2605_23945_b200/libtpshift_b200.so
python -c "
import json
for n in ('sb_st3','sb_st2'):
    d=json.load(open('gpurun_out/'+n+'.json')); print(n, round(d['generation_time'],3))"
