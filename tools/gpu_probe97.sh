for c in 64 504; do timeout 300 python tools/trace_prefill.py qwen2.5-7b $c 2>&1 | head -6; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
