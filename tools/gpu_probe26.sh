timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048
timeout 300 python tools/trace_step.py qwen2.5-7b 1 1 2048
timeout 300 python tools/trace_step.py qwen2.5-7b 1 64 2048
