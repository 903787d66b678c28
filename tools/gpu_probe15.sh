timeout 600 python tools/solo_step.py qwen2.5-7b 1,2,8 1,16,64 2048 ";fuse_push" 2>&1 | grep -v watchdog
