#!/bin/bash
# ncu evidence for the factored kernels (full-size b/m3/exp1 and c/m5/exp1
# sweeps) and the launch list of the default bench command.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$B > gpurun_out/plain_launch_f.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_factored.csv $B > gpurun_out/ncu_launch_f.log 2>&1
P="python tools/prof_sweep.py --workload b/m3/exp1 --full --reps 2 --algorithm factored"
$P > gpurun_out/plain_pf.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_b_fact -s 2 -c 2 \
      -o gpurun_out/k1b_factored $P > gpurun_out/ncu_pf.log 2>&1
C="python tools/prof_sweep.py --workload c/m5/exp1 --full --reps 2 --algorithm factored"
$C > gpurun_out/plain_cf.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_c_fact -s 2 -c 2 \
      -o gpurun_out/k1c_factored $C > gpurun_out/ncu_cf.log 2>&1
ls gpurun_out
