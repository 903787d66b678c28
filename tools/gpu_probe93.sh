timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "grouped_prefill or qkv_rope_in_kernel" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in 64 256 504; do timeout 300 python tools/trace_prefill.py qwen2.5-7b $c 2>&1 | head -8; done
