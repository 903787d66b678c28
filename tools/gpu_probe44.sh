for b in 16 48; do timeout 300 python tools/trace_step.py qwen2.5-7b 8 $b 3072 2>&1 | sed -n 1,12p; done
timeout 300 python tools/trace_step.py qwen2.5-7b 8 16 3072 2>&1 | sed -n 13,26p
