"""Factored b/m3/exp1 sweep: K1 time (measurement hook, 10 reps), hash of V'
+ actions, max |dV| against a reference run, and the converged solve."""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("b/m3/exp1").set_algorithm("factored")
n = m.state_count()
V = np.random.default_rng(3).uniform(-20.0, 20.0, n)
P.bellman_backup_batch(m, V, 0, n)
P.profile_enable(True)
reps = 10
for _ in range(reps):
    v, a = P.bellman_backup_batch(m, V, 0, n)
ms, kl, al = P.profile_read()
P.profile_enable(False)
h = hashlib.sha256(v.tobytes() + a.tobytes()).hexdigest()[:16]
ref = os.environ.get("REF")
extra = ""
if ref and os.path.exists(ref):
    z = np.load(ref)
    extra = f" max|dV| {np.max(np.abs(v - z['v'])):.3e} act diffs {int(np.sum(a != z['a']))}"
elif ref:
    np.savez(ref, v=v, a=a)
t = time.perf_counter()
r = P.run_value_iteration(m)
w = time.perf_counter() - t
print(f"b/m3/exp1 K1 {ms / reps:.3f} ms/sweep hash {h}{extra} | solve {r.iterations} it {r.wall_seconds:.4f} s")
