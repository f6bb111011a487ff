# A/B of one env switch on the default bench step (+ optional test file):
#   VAR=PVI_E2E_PAIRS VALS="0 1" TESTVALS=1 TESTS=tests/test_gpu_factored.py bash tools/gpu/env_ab.sh
mkdir -p gpurun_out
B="python bench.py --no-alt --no-simopt --no-solve --no-cpu-baseline --steps 10 ${EXTRA:-}"
for v in $VALS; do env $VAR=$v timeout 300 $B > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err; done
for v in $VALS; do
python - $v <<'P'
import json, sys
v=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, "step %.3f ms" % d["ms_per_step"], "kernel %.3f" % d["roofline"]["kernel_ms_per_launch"],
          "e2e %.3f ms" % (1e3 * d["config"]["terms_per_sweep"] / d["e2e"]["value"]) if "e2e" in d else "", d["clocks"]["sm_mhz"])
except Exception as e:
    print(v, "failed", e, open(f"gpurun_out/ab_{v}.err").read()[-2000:])
P
done
for v in ${TESTVALS:-}; do env $VAR=$v timeout 600 python -m pytest ${TESTS:-tests/test_gpu_factored.py} -x -q 2>&1 | tail -2; done
