"""Run the device backup over a slice of a preset's states (for ncu captures).

  python tools/prof_sweep.py --workload b/m3/exp1 --frac 0.015625 --reps 2
The slice starts mid-space so its per-state cost is representative."""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="b/m3/exp1")
ap.add_argument("--frac", type=float, default=1 / 64)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--precision", default="f64")
ap.add_argument("--algorithm", default="exact")
ap.add_argument("--full", action="store_true", help="sweep all states")
a = ap.parse_args()
m = P.make_preset(a.workload).set_algorithm(a.algorithm)
n = m.state_count()
cnt = max(1, int(n * a.frac))
lo = 0 if a.full else (n // 2) // 4096 * 4096
hi = n if a.full else min(n, lo + cnt)
V = m.initial_values().astype(np.float32 if a.precision == "f32" else np.float64)
for r in range(a.reps):
    t = time.perf_counter()
    P.bellman_backup_batch(m, V, lo, hi, precision=a.precision)
    print(f"rep {r}: states [{lo},{hi}) {time.perf_counter() - t:.4f} s")
