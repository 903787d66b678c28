timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -2
for e in 1 0; do TPS_ATTN_EARLY=$e timeout 600 python tools/solo_step.py qwen2.5-7b 4,8 1,2,8 2048 2>&1 | grep -v watchdog; done
TPS_ATTN_EARLY=1 timeout 600 python tools/solo_step.py qwen2.5-7b 8 1 8192 2>&1 | grep -v watchdog
TPS_ATTN_EARLY=0 timeout 600 python tools/solo_step.py qwen2.5-7b 8 1 8192 2>&1 | grep -v watchdog
