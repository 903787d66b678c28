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
