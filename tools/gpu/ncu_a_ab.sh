# k_a_fact_* time / instructions: current build vs lib/libpvi_b200_old.so (W=a/m5/exp5 or exp6)
C="tools/prof_sweep.py --workload ${W:-a/m5/exp5} --full --reps 3 --algorithm factored"
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
ncu --metrics $M --clock-control none -k regex:k_a_fact --csv python $C > gpurun_out/a_new.csv 2>&1
ncu --metrics $M --clock-control none -k regex:k_a_fact --csv python tools/with_lib.py paper_2303_10672_b200/lib/libpvi_b200_old.so $C > gpurun_out/a_old.csv 2>&1
echo new; python tools/ncu_brief.py gpurun_out/a_new.csv; echo old; python tools/ncu_brief.py gpurun_out/a_old.csv
