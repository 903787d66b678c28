set -x
mkdir -p gpurun_out
free -g | head -2; nproc
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_swapab -s 8 -c 4 -o gpurun_out/ncu_gemm_families python tools/ncu_gemm_traffic.py 64 > gpurun_out/ncu_gemm.log 2>&1; tail -2 gpurun_out/ncu_gemm.log
ncu -i gpurun_out/ncu_gemm_families.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/ncu_gemm_families.csv 2>&1
python tools/ncu_gemm_traffic.py --summarise gpurun_out/ncu_gemm_families.csv 64 | tail -5
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -c 6000 gpurun_out/bench.log
