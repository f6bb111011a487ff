#!/bin/bash
# ncu evidence for the factored kernels (full-size b/m3/exp1, c/m5/exp1 and
# c/m5/exp2 sweeps) and the launch list of the default bench command.  Each
# ncu command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$B > gpurun_out/plain_launch_f.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_factored.csv $B > gpurun_out/ncu_launch_f.log 2>&1
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$P > gpurun_out/plain_pf.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_b_fact -s 2 -c 2 \
      -o gpurun_out/k1b_factored $P > gpurun_out/ncu_pf.log 2>&1
for W in c/m5/exp1 c/m5/exp2; do
  T=$(echo $W | tr '/' '_')
  C="python tools/prof_sweep.py --workload $W --full --reps 2 --algorithm factored"
  $C > gpurun_out/plain_$T.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k_c_ -s 0 -c 12 \
        -o gpurun_out/k1c_$T $C > gpurun_out/ncu_$T.log 2>&1
done
ls gpurun_out
# summaries (the raw reports are large): keep the JSON digests and SASS/source
# pages of the top kernels, drop the .ncu-rep files unless KEEP_REPORTS=1
python tools/ncu_summary.py --launches gpurun_out/launches_factored.csv gpurun_out/launch_list_factored.json
for R in k1b_factored k1c_c_m5_exp1 k1c_c_m5_exp2; do
  [ -f gpurun_out/$R.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$R.ncu-rep gpurun_out/${R}_ncu.json
done
[ -f gpurun_out/k1b_factored.ncu-rep ] && ncu -i gpurun_out/k1b_factored.ncu-rep --page source --csv --print-source sass > gpurun_out/k1b_factored_sass.csv 2>/dev/null
[ "${KEEP_REPORTS:-0}" = "1" ] || rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
