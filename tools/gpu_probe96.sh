timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "grouped_prefill" 2>&1 | tail -2
for c in 64 504; do timeout 300 python tools/trace_prefill.py qwen2.5-7b $c 2>&1 | head -5; done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
