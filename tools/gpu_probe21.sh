timeout 600 python tools/gemm_mix.py qwen2.5-7b 2,8 1 2>&1 | grep chain
timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16,64 2048 ";fuse_push" 2>&1 | grep -v watchdog
