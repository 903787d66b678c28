timeout 300 python tools/qkv_probe.py
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "qkv_rope_in_kernel" 2>&1 | tail -2
