python - <<'P'
import sys, time, tempfile, os
sys.path.insert(0, ".")
from paper_2303_10672_b200 import runner
for preset in ["b/m3/exp1", "c/m5/exp1", "a/m5/exp5"]:
    with tempfile.TemporaryDirectory() as d:
        t = time.perf_counter()
        out = runner.cmd_solve(preset, d, algorithm=os.environ.get("ALGO", "exact"))
        t1 = time.perf_counter()
        runner.cmd_evaluate(preset, d, vi_policy=os.path.join(d, "policy.csv"), n_rollouts=10000)
        t2 = time.perf_counter()
        sizes = {f: os.path.getsize(os.path.join(d, f)) for f in os.listdir(d)}
        print(preset, f"cmd_solve {t1 - t:.2f} s (iterations {out.iterations}), cmd_evaluate {t2 - t1:.2f} s", sizes, flush=True)
P
