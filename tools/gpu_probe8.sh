mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k push > gpurun_out/push_test.log 2>&1; tail -3 gpurun_out/push_test.log
for tp in 2 4 8; do timeout 300 python tools/tp_step.py qwen2.5-7b $tp 1,16,64 2048 >> gpurun_out/tp_step.log 2>&1; done
cat gpurun_out/tp_step.log
