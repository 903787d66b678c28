timeout 900 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -3
timeout 900 python tools/solo_step.py qwen2.5-7b 1,8 1,16,64 2048 ";+fuse_rope" 2>&1 | grep -v watchdog
timeout 600 python tools/solo_step.py qwen2.5-7b 1 64 6144 ";+fuse_rope" 2>&1 | grep -v watchdog
