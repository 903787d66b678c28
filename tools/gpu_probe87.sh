for c in 64 256 504; do timeout 300 python tools/trace_prefill.py qwen2.5-7b $c 2>&1 | head -12; done
