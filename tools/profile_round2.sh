#!/bin/bash
# Round-2 ncu evidence (run on the GPU box, one GPU):
#  1. launch list of the default bench step (b/m3/exp1, factored);
#  2. --set full of both stages of one full-size b/m3/exp1 factored sweep
#     (k_b_fact_w16p, k_b_fact_qw4 with its TMEM running maxima);
#  3. --set full of one c/m5/exp2 and one c/m5/exp1 factored sweep (weekday
#     tables: k_c_fact_g, k_c_bin_tile_p x3, k_c_bin_qf / k_c_bin_q);
#  4. --set full of the rollout kernel on a simopt-sized batch (50 x 4096).
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt --no-others"
$B > gpurun_out/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r2_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt --no-others"
$P > gpurun_out/plain_pf.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_b_fact -s 2 -c 2 \
      -o gpurun_out/r2_k1b $P > gpurun_out/ncu_pf.log 2>&1
for W in c/m5/exp1 c/m5/exp2; do
  T=$(echo $W | tr '/' '_')
  C="python tools/prof_sweep.py --workload $W --full --reps 2 --algorithm factored"
  $C > gpurun_out/plain_$T.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k_c_ -s 5 -c 5 \
        -o gpurun_out/r2_k1c_$T $C > gpurun_out/ncu_$T.log 2>&1
done
S="python tools/sim_batch.py"
$S > gpurun_out/plain_sim.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_rollouts -s 1 -c 1 \
      -o gpurun_out/r2_k5 $S > gpurun_out/ncu_sim.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/r2_launches.csv gpurun_out/r2_launch_list.json
for R in r2_k1b r2_k1c_c_m5_exp1 r2_k1c_c_m5_exp2 r2_k5; do
  [ -f gpurun_out/$R.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$R.ncu-rep gpurun_out/${R}_ncu.json
done
[ "${KEEP_REPORTS:-0}" = "1" ] || rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
