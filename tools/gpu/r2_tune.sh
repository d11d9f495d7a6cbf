# round-2 tuning sweeps (tools only): PP layout/occupancy variants, bit-identity required
mkdir -p gpurun_out
tools/pp_tune > gpurun_out/pp_tune.txt 2>&1
tools/acc_tune > gpurun_out/acc_tune.txt 2>&1
cat gpurun_out/pp_tune.txt gpurun_out/acc_tune.txt
