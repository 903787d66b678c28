timeout 600 python -m pytest tests/test_gpu_kernels.py -q -k "grouped_prefill" 2>&1 | tail -3
for c in 64 504; do timeout 300 python tools/trace_prefill.py qwen2.5-7b $c 2>&1 | head -8; done
timeout 600 python tools/trace_prefill.py mini-llama 256 2>&1 | head -3
