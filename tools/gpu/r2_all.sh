bash tools/gpu/r2_tune.sh
bash tools/gpu/r2_check.sh
