timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/trace_step.py qwen2.5-7b 8 1 2048 2>&1 | head -12
timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16,64 2048 "" 2>&1 | grep -v watchdog
