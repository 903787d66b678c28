timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_multiprocess.py -x -q 2>&1 | tail -2
bash tools/gpu_profile.sh
timeout 1500 python tools/profile_b200.py --model qwen2.5-32b --token-cap 262144 --budget 1200 --out gpurun_out/b200_qwen2.5-32b.csv > gpurun_out/profile_q32.log 2>&1
tail -1 gpurun_out/profile_q32.log
