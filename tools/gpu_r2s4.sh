# Round 2, session 4 (GPU reopened): validate the GEMV and the post-closure changes first, then measure.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
# first contact under memcheck: an out-of-bounds access is reported by the instrumentation instead
# of faulting the device (the kernel-level tests only; the step tests follow without the tool)
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_tail_gemv.py -x -q \
  -k "not full_shapes and not decode and not graph" > gpurun_out/memcheck_gemv.log 2>&1; tail -5 gpurun_out/memcheck_gemv.log
grep -q "ERROR SUMMARY: 0 errors" gpurun_out/memcheck_gemv.log || { echo "memcheck not clean: stop"; exit 1; }
timeout 900 python -m pytest tests/test_gpu_tail_gemv.py -x -q -k "not full_shapes" > gpurun_out/pytest_gemv.log 2>&1; tail -5 gpurun_out/pytest_gemv.log
for g in 0 4; do echo "TPS_GEMV_ROWS=$g"; TPS_GEMV_ROWS=$g timeout 600 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,2,4 2048 2>&1 | grep step; done
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; tail -c 6000 gpurun_out/bench.log
TPS_GEMV_ROWS=4 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemv_kernel -s 20 -c 8 -o gpurun_out/ncu_gemv python tools/solo_step.py qwen2.5-7b 8 1 2048 > gpurun_out/ncu_gemv.log 2>&1
ncu -i gpurun_out/ncu_gemv.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size > gpurun_out/ncu_gemv.csv 2>&1; head -12 gpurun_out/ncu_gemv.csv
