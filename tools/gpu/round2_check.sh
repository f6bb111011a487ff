python -m pytest tests -m gpu -q > gpurun_out/t8.log 2>&1; tail -3 gpurun_out/t8.log
C="python tools/prof_sweep.py --workload c/m5/exp2 --full --reps 2 --algorithm factored"
$C > gpurun_out/plain_c8.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_c_bin -s 4 -c 4 -o gpurun_out/r2_diag $C > gpurun_out/ncu_c8.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_diag.ncu-rep gpurun_out/r2_k1c_diag_exp2_ncu.json
ncu -i gpurun_out/r2_diag.ncu-rep --page source --csv --print-source sass -k regex:k_c_bin_diag > gpurun_out/r2_diag_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err; tail -c 600 gpurun_out/bench8.json
