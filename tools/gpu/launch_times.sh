# per-kernel durations (ncu launch list) of the bench step under env settings
mkdir -p gpurun_out
P="python bench.py --steps 1 --warmup 3 --no-solve --no-e2e --no-cpu-baseline --no-alt --no-simopt ${EXTRA:-}"
for v in $VALS; do
  env $VAR=$v $P > gpurun_out/lt_plain_$v.log 2>&1 && \
  env $VAR=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lt_$v.csv $P > /dev/null 2>&1
  python - $v <<'Q'
import csv, sys, collections, re
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/lt_{v}.csv")) if len(r) > 10]
h = rows[0]; ik = h.index("Kernel Name"); im = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    m = re.search(r"(k_\w+|\w*elementwise\w*)", r[ik]); agg[m.group(1) if m else r[ik][:30]].append(float(r[im]))
for k, xs in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(v, f"{k:28s} n={len(xs):3d} last={xs[-1]:10.1f} min={min(xs):10.1f}")
Q
done
