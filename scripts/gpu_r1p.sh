bash scripts/gpu_scale.sh
bash scripts/gpu_profile.sh r1p tests 150
