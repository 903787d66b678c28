for c in 2048 6144; do timeout 300 python tools/trace_step.py qwen2.5-7b 1 64 $c 2>&1 | head -14; done
timeout 300 python tools/trace_step.py qwen2.5-7b 1 16 4096 2>&1 | head -14
