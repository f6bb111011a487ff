#!/bin/bash
# ncu evidence for the current default bench path (run on the GPU box):
#  1. launch list (gpu__time_duration per launch) of the bench command
#  2. one --set full capture of each factored-B kernel at full size
#     (stage 2 k_b_fact_qw4, stage 1 k_b_fact_w16p), summarised to JSON,
#     plus the stage-2 SASS source page with per-instruction stall samples.
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r1b}
B="python bench.py --steps 2 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$B > gpurun_out/${TAG}_plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$P > gpurun_out/${TAG}_plain_full.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_b_fact_(qw4|w16p)" -s 2 -c 2 \
      -o gpurun_out/${TAG}_k1b $P > gpurun_out/${TAG}_ncu_full.log 2>&1
python tools/ncu_summary.py --launches gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_launch_list.json
python tools/ncu_summary.py gpurun_out/${TAG}_k1b.ncu-rep gpurun_out/${TAG}_k1b_ncu.json
ncu -i gpurun_out/${TAG}_k1b.ncu-rep --page source --csv --print-source sass -k regex:qw4 > gpurun_out/${TAG}_qw4_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
