mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16,64 2048 ";fuse_push" 2>&1 | grep -v watchdog
timeout 900 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; tail -c 1500 gpurun_out/bench.log
