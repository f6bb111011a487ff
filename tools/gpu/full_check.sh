# round-end style check on one GPU: the whole -m gpu suite, smoke(), the
# default bench line (+ c/m5 launch lists for the C numbers)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/full_t.log 2>&1; tail -3 gpurun_out/full_t.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/full_smoke.log 2>&1; tail -1 gpurun_out/full_smoke.log
python bench.py > gpurun_out/full_bench.json 2> gpurun_out/full_bench.err; tail -c 300 gpurun_out/full_bench.json
for W in c/m5/exp1 c/m5/exp2; do
  T=$(echo $W | tr '/' '_')
  ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_c_ \
      --log-file gpurun_out/r2_c_launches_$T.csv python tools/prof_sweep.py --workload $W --full --reps 2 --algorithm factored > /dev/null 2>&1
done
