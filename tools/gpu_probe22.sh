timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/gemm_mix.py qwen2.5-7b 2,8 1 2>&1 | grep chain
timeout 900 python tools/solo_step.py qwen2.5-7b 2,8 1,16 2048 ";fuse_push" 2>&1 | grep -v watchdog
