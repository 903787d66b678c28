mkdir -p gpurun_out
timeout 1200 python tools/profile_b200.py --model llama3-8b --budget 900 --out gpurun_out/b200_llama3-8b.csv > gpurun_out/profile_llama.log 2>&1
tail -2 gpurun_out/profile_llama.log
timeout 1500 python tools/profile_b200.py --model qwen2.5-32b --token-cap 262144 --budget 1200 --out gpurun_out/b200_qwen2.5-32b.csv > gpurun_out/profile_q32.log 2>&1
tail -2 gpurun_out/profile_q32.log
