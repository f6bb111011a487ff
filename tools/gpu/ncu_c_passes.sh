# per-launch time / DRAM / instructions of one c/m5/exp2 factored sweep
C="python tools/prof_sweep.py --workload ${W:-c/m5/exp2} --full --reps 1 --algorithm factored"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_c_ -c ${N:-5} --csv $C > gpurun_out/ncu_c_passes.csv 2>&1
python tools/ncu_brief.py gpurun_out/ncu_c_passes.csv
