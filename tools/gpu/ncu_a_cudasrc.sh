# per-CUDA-line attribution of a factored A sweep kernel (W=a/m5/exp5|exp6)
set -u
mkdir -p gpurun_out
C="python tools/prof_sweep.py --workload ${W:-a/m5/exp6} --full --reps 3 --algorithm factored"
T=${TAG:-afl}
ncu --set full --clock-control none --import-source on -k regex:k_a_fact -s 1 -c 1 -o gpurun_out/$T $C > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_cuda.csv 2>&1
rm -f gpurun_out/$T.ncu-rep
