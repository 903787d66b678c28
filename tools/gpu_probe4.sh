mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for ctx in 512 4096; do timeout 300 python tools/skip_probe.py qwen2.5-7b 1,16,64 $ctx >> gpurun_out/skip_probe2.log 2>&1; done
timeout 600 python tools/switch_bench.py --world 2 --pairs 1:2,2:1 --samples 16 --ctx 4096 > gpurun_out/switch_bench.log 2>&1
timeout 600 python tools/switch_bench.py --world 4 --pairs 1:4,2:4 --samples 16 --ctx 2048 --modes 0 >> gpurun_out/switch_bench.log 2>&1
tail -3 gpurun_out/switch_bench.log
