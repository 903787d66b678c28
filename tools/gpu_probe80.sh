timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16,64 2048 "+silu_fused;+silu_unfused" 2>&1 | grep -v watchdog
