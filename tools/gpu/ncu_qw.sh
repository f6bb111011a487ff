#!/bin/bash
# ncu full capture of the factored-B stage-2 kernel (one launch, full size)
# plus its SASS source page with per-instruction stall samples.
set -u
mkdir -p gpurun_out
K=${K:-k_b_fact_qw4}
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$P > gpurun_out/plain_q.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o gpurun_out/$K $P > gpurun_out/ncu_q.log 2>&1
python tools/ncu_summary.py gpurun_out/$K.ncu-rep gpurun_out/${K}_ncu.json
ncu -i gpurun_out/$K.ncu-rep --page source --csv --print-source sass > gpurun_out/${K}_sass.csv 2>/dev/null
ncu -i gpurun_out/$K.ncu-rep --page details --csv > gpurun_out/${K}_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
