bash tools/gpu_profile.sh
bash tools/gpu_final.sh
