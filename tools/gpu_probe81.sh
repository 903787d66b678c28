timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/solo_step.py qwen2.5-7b 2,4,8 1,8,12,16,32,64 3072 "" 2>&1 | grep -v watchdog
