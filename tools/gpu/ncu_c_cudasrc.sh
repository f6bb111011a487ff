# per-CUDA-source-line instruction counts of one c/m5 kernel (K=<regex>, W=<workload>)
set -u
mkdir -p gpurun_out
C="python tools/prof_sweep.py --workload ${W:-c/m5/exp2} --full --reps 2 --algorithm factored"
T=${TAG:-c_cudasrc}
ncu --set full --clock-control none --import-source on -k regex:${K} -s 1 -c 1 -o gpurun_out/$T $C > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_cuda.csv 2>&1
rm -f gpurun_out/$T.ncu-rep
