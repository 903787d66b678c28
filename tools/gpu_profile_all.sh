bash tools/gpu_profile.sh
bash tools/gpu_profile2.sh
