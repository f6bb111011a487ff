# --set full + source page of the rollout kernel on a simopt-sized batch (b/m2/exp1)
mkdir -p gpurun_out
S="python tools/sim_batch.py"
$S > gpurun_out/plain_sim.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_rollouts -s 1 -c 1 -o gpurun_out/r2_k5b $S > gpurun_out/ncu_k5.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_k5b.ncu-rep gpurun_out/r2_k5b_ncu.json
ncu -i gpurun_out/r2_k5b.ncu-rep --page source --csv > gpurun_out/r2_k5b_src.csv 2>&1
ncu -i gpurun_out/r2_k5b.ncu-rep --page source --csv --print-source cuda > gpurun_out/r2_k5b_cuda.csv 2>&1
rm -f gpurun_out/*.ncu-rep
python tools/ncu_src_hot.py gpurun_out/r2_k5b_src.csv 16
