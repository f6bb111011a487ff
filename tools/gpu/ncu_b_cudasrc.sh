# per-CUDA-source-line instruction counts of one factored b/m3/exp1 kernel (K=<regex>)
set -u
mkdir -p gpurun_out
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt --no-others"
T=${TAG:-b_cudasrc}
ncu --set full --clock-control none --import-source on -k regex:${K} -s 2 -c 1 -o gpurun_out/$T $P > gpurun_out/ncu_$T.log 2>&1
ncu -i gpurun_out/$T.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_cuda.csv 2>&1
rm -f gpurun_out/$T.ncu-rep
