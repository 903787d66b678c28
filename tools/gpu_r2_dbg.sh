timeout 600 python -m pytest tests/test_gpu_persist.py tests/test_gpu_decode.py -x -q 2>&1 | grep -v "^tps watchdog" | tail -2
timeout 900 python -m pytest tests/test_gpu_decode_fullshape.py -x -q -k "persist_batch16 or True" 2>&1 | tail -2
