timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for sm in 1 0; do
TPS_GEMM_SMALL=$sm timeout 600 python tools/gemm_mix.py qwen2.5-7b 1,8 1 2>&1 | grep chain | sed "s/^/small=$sm /"
TPS_GEMM_SMALL=$sm timeout 900 python tools/solo_step.py qwen2.5-7b 1,2,4,8 1,16 2048 "" 2>&1 | grep -v watchdog | sed "s/^/small=$sm /"
done
