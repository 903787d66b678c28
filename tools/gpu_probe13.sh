mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16,64 2048 ";fuse_push;attention,qkv_rope" 2>&1 | grep -v watchdog
