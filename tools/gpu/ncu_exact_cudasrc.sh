# per-CUDA-line attribution of an exact sweep kernel (K=<regex>, W=<workload>, a 1/64 slice)
set -u
mkdir -p gpurun_out
C="python tools/prof_sweep.py --workload ${W:-b/m3/exp1} --frac 0.015625 --reps 2 --algorithm exact"
T=${TAG:-ex}
ncu --set full --clock-control none --import-source on -k regex:${K} -s 1 -c 1 -o gpurun_out/$T $C > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_cuda.csv 2>&1
rm -f gpurun_out/$T.ncu-rep
