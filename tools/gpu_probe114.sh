for tp in 1 8; do timeout 300 python tools/trace_prefill.py qwen2.5-7b 64 $tp 2>&1 | head -12; done
