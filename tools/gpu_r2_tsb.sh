for cfg in "8 32 2 2" "8 32 4 2" "16 16 4 2" "16 16 3 2" "8 16 8 2" "16 8 8 2" "32 8 4 2" "128 1 8 0"; do ./tools/cuda/tsb $cfg; done
