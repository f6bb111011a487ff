# --set full of one kernel of a c/m5 factored sweep: K=<kernel regex> W=<workload>
set -u
mkdir -p gpurun_out
C="python tools/prof_sweep.py --workload ${W:-c/m5/exp2} --full --reps 2 --algorithm factored"
T=${TAG:-c_full}
$C > gpurun_out/plain_$T.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K} -s 1 -c 1 -o gpurun_out/$T $C > gpurun_out/ncu_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/$T.ncu-rep gpurun_out/${T}_ncu.json
ncu -i gpurun_out/$T.ncu-rep --page source --csv > gpurun_out/${T}_src.csv 2>&1
ncu -i gpurun_out/$T.ncu-rep --page details --csv > gpurun_out/${T}_details.csv 2>&1
rm -f gpurun_out/$T.ncu-rep
