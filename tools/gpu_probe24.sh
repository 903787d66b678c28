timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,4,16 2048 ";+fuse_rope" 2>&1 | grep -v watchdog | sed 's/^/minbal64 /'
TPS_ATTN_MIN_BAL=1 timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,4,16 2048 ";+fuse_rope" 2>&1 | grep -v watchdog | sed 's/^/minbal1 /'
