TPS_ATTN_MAX_CLUSTER=0 timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048 2>&1 | head -22
TPS_ATTN_EARLY=0 timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048 2>&1 | head -2
