# Everything this session could not run while gpurun was closed (validation first).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -c 6000 gpurun_out/bench.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_swapab -s 8 -c 4 -o gpurun_out/ncu_gemm_families python tools/ncu_gemm_traffic.py 64 > gpurun_out/ncu_gemm.log 2>&1
ncu -i gpurun_out/ncu_gemm_families.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/ncu_gemm_families.csv 2>&1
python tools/ncu_gemm_traffic.py --summarise gpurun_out/ncu_gemm_families.csv 64 | tail -3
for t in memcheck racecheck synccheck; do timeout 900 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_stage.py > gpurun_out/sanitizer_$t.log 2>&1; tail -3 gpurun_out/sanitizer_$t.log; done
timeout 1500 python bench.py --model llama3-8b --per-gpu-batch 32 --l-max 16384 --no-cpu --no-switch --no-tail --steps 1 --warmup 1 > gpurun_out/bench_c3_n1.log 2>&1; tail -c 1500 gpurun_out/bench_c3_n1.log
timeout 1500 python bench.py --virtual 4 --alias-replicas --model qwen2.5-32b --initial-tp 2 --tp-list 2,4 --per-gpu-batch 2 --l-max 4096 --static-tps "" --no-e2e --steps 1 --warmup 1 > gpurun_out/bench_c4_virtual.log 2>&1; tail -c 1500 gpurun_out/bench_c4_virtual.log
TPS_SHARE_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29731 bench.py --gpus 2 --steps 1 --warmup 1 --per-gpu-batch 16 --l-max 2048 > gpurun_out/bench_n2_shared.log 2>&1; tail -c 1500 gpurun_out/bench_n2_shared.log
timeout 2400 python tools/switch_bench.py --models llama3-8b,qwen2.5-32b --worlds 2,4,8 --samples 1,16 --ctx 4096,16384 > gpurun_out/switch_sweep_8b_32b.log 2>&1; grep -c copy_kernel_ms gpurun_out/switch_sweep_8b_32b.log
