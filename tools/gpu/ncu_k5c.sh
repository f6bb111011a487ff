set -u
mkdir -p gpurun_out
S="python ${SCRIPT:-tools/sim_batch_c.py}"
ncu --set full --clock-control none --import-source on -k regex:k_rollouts -s 1 -c 1 -o gpurun_out/k5c $S > gpurun_out/ncu_k5c.log 2>&1
ncu -i gpurun_out/k5c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k5c_cuda.csv 2>&1
rm -f gpurun_out/*.ncu-rep
