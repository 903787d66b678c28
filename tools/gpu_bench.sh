mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -c 3000 gpurun_out/bench.log
timeout 600 python tools/switch_bench.py --world 2 --pairs 1:2 --samples 16 --ctx 4096 --modes 0,1 > gpurun_out/switch_bench.log 2>&1
timeout 600 python tools/switch_bench.py --world 4 --model llama3-8b --pairs 1:4,2:4,4:2 --samples 16 --ctx 4096 --modes 1 >> gpurun_out/switch_bench.log 2>&1
cat gpurun_out/switch_bench.log
