mkdir -p gpurun_out
B="python bench.py --no-alt --no-simopt --no-solve --no-e2e --no-cpu-baseline --steps 10"
MODES=${MODES:-"0 1 3"}
for v in $MODES; do PVI_B_QW4=$v timeout 300 $B > gpurun_out/qw4_$v.json 2>gpurun_out/qw4_$v.err; done
for v in $MODES; do
python - $v <<'P'
import json, sys
v=sys.argv[1]
d=json.loads(open(f"gpurun_out/qw4_{v}.json").read().strip().splitlines()[-1])
print(v, d["ms_per_step"], d["roofline"]["kernel_ms_per_launch"], d["clocks"]["sm_mhz"])
P
done
for v in ${TESTMODES:-}; do PVI_B_QW4=$v timeout 600 python -m pytest tests/test_gpu_factored.py -x -q 2>&1 | tail -1; done
