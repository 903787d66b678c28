timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048 2>&1 | head -22
