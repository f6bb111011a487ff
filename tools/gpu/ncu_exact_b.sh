mkdir -p gpurun_out
P="python bench.py --algorithm exact --steps 1 --warmup 1 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt"
$P > gpurun_out/plain_eb.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_b_geo -s 1 -c 1 \
      -o gpurun_out/eb $P > gpurun_out/ncu_eb.log 2>&1
python tools/ncu_summary.py gpurun_out/eb.ncu-rep gpurun_out/r1b_k1b_exact_ncu.json
ncu -i gpurun_out/eb.ncu-rep --page source --csv --print-source sass > gpurun_out/eb_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
