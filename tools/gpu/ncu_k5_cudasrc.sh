# per-CUDA-line attribution of the rollout kernel (b/m2/exp1 simopt-sized batch) and the A LIFO sweep
set -u
mkdir -p gpurun_out
S="python tools/sim_batch.py"
ncu --set full --clock-control none --import-source on -k regex:k_rollouts -s 1 -c 1 -o gpurun_out/k5l $S > gpurun_out/ncu_k5l.log 2>&1
ncu -i gpurun_out/k5l.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k5l_cuda.csv 2>&1
C="python tools/prof_sweep.py --workload a/m5/exp5 --full --reps 3 --algorithm factored"
ncu --set full --clock-control none --import-source on -k regex:k_a_fact -s 1 -c 1 -o gpurun_out/al $C > gpurun_out/ncu_al.log 2>&1
ncu -i gpurun_out/al.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/al_cuda.csv 2>&1
rm -f gpurun_out/*.ncu-rep
