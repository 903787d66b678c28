set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_switch_items.py tests/test_gpu_reshard_fullsize.py tests/test_gpu_coordinator.py tests/test_gpu_multiprocess.py -x -q > gpurun_out/pytest_switch.log 2>&1; tail -15 gpurun_out/pytest_switch.log
timeout 1200 python tools/switch_bench.py --worlds 2,4,8 --samples 16 --ctx 4096 > gpurun_out/switch_sweep_a.log 2>&1; grep -v watchdog gpurun_out/switch_sweep_a.log | tail -30
