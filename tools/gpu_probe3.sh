mkdir -p gpurun_out
for ctx in 512 4096; do timeout 300 python tools/skip_probe.py qwen2.5-7b 1,16,64 $ctx >> gpurun_out/skip_probe.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_multiprocess.py -x -q > gpurun_out/mp_test.log 2>&1
tail -5 gpurun_out/mp_test.log
