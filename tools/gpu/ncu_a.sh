# a/m5/exp5 factored: launch list of a short solve and --set full of the LIFO kernel
mkdir -p gpurun_out
C="python tools/prof_sweep.py --workload a/m5/exp5 --full --reps 3 --algorithm factored"
$C > gpurun_out/plain_a.log 2>&1
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_bytes.sum --clock-control none --csv $C > gpurun_out/ncu_a_launch.csv 2>&1
python tools/ncu_brief.py gpurun_out/ncu_a_launch.csv | tail -12
ncu --set full --clock-control none --import-source on -k regex:k_a_fact -s 2 -c 1 -o gpurun_out/r2_a_lifo $C > gpurun_out/ncu_a.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_a_lifo.ncu-rep gpurun_out/r2_a_lifo_ncu.json
ncu -i gpurun_out/r2_a_lifo.ncu-rep --page source --csv > gpurun_out/r2_a_lifo_src.csv 2>&1
ncu -i gpurun_out/r2_a_lifo.ncu-rep --page details --csv > gpurun_out/r2_a_lifo_details.csv 2>&1
rm -f gpurun_out/*.ncu-rep
