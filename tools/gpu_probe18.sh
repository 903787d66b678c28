timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1 2048 ";qkv_rope;attention;add_norm;silu;qkv_rope,attention,add_norm,silu;linear;fuse_push" 2>&1 | grep -v watchdog
TPS_ATTN_MIN_BAL=1 timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,4,16 2048 ";attention" 2>&1 | grep -v watchdog | sed 's/^/minbal1 /'
timeout 900 python tools/solo_step.py qwen2.5-7b 8 4,16 2048 ";attention" 2>&1 | grep -v watchdog | sed 's/^/default /'
