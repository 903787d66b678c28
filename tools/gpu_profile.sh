mkdir -p gpurun_out
timeout 1500 python tools/profile_b200.py --model qwen2.5-7b --budget 1200 --out gpurun_out/b200_qwen2.5-7b.csv > gpurun_out/profile.log 2>&1
tail -5 gpurun_out/profile.log; grep -c . gpurun_out/b200_qwen2.5-7b.csv
