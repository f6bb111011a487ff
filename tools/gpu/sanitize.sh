#!/bin/bash
# compute-sanitizer over the factored sweeps.  Run on the
# GPU box: bash tools/gpu/sanitize.sh ; logs in gpurun_out/sanitize/.
set -u
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for c in b_m2 c_m3_exp1 c_m3_exp2 a_m4_fifo a_m4_lifo b_m3_slice; do
  python tools/sanitize_sweeps.py $c > gpurun_out/sanitize/plain_$c.log 2>&1 || { echo "plain $c failed"; continue; }
  for t in memcheck racecheck synccheck initcheck; do
    extra=""
    [ $t = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $t $extra --error-exitcode 99 --print-limit 50 \
      python tools/sanitize_sweeps.py $c > gpurun_out/sanitize/${t}_$c.log 2>&1
    echo "$t $c exit=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
