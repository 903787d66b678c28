mkdir -p gpurun_out
timeout 1200 python tools/profile_b200.py --model llama3-8b --budget 900 --out gpurun_out/b200_llama3-8b.csv > gpurun_out/profile_llama.log 2>&1
tail -1 gpurun_out/profile_llama.log
