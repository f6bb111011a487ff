#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command, one full
# ncu capture of the headline K1-B sweep at full size, one of K1-C on a
# c/m5 slice.  Each ncu command runs only after the same command exited 0.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-solve --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
P="python bench.py --steps 1 --warmup 1 --no-solve --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_b_geo -s 1 -c 1 \
      -o gpurun_out/k1b_full $P > gpurun_out/ncu_full.log 2>&1
C="python tools/prof_sweep.py --workload c/m5/exp1 --frac 0.02 --reps 2"
$C > gpurun_out/plain_c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_c -s 1 -c 1 \
      -o gpurun_out/k1c_slice $C > gpurun_out/ncu_c.log 2>&1
ls -la gpurun_out
