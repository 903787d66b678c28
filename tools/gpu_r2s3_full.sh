set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -c 2500 gpurun_out/bench.log
timeout 2400 python tools/switch_bench.py --worlds 2,4,8 --samples 1,16,64 --ctx 4096,16384 > gpurun_out/switch_sweep_7b.log 2>&1; grep -c copy_kernel_ms gpurun_out/switch_sweep_7b.log
