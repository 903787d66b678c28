set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 4000 gpurun_out/bench.log
timeout 600 python tools/solo_step.py qwen2.5-7b 1,8 1,16 2048 > gpurun_out/solo_base.log 2>&1; grep -v watchdog gpurun_out/solo_base.log | tail -8
TPS_PERSIST=1 timeout 600 python tools/solo_step.py qwen2.5-7b 1,8 1,16 2048 > gpurun_out/solo_persist.log 2>&1; grep -v watchdog gpurun_out/solo_persist.log | tail -8
TPS_PERSIST=1 timeout 300 python tools/persist_trace.py qwen2.5-7b 8 1 2048 > gpurun_out/persist_trace.log 2>&1; tail -40 gpurun_out/persist_trace.log
