"""Factored A sweeps (a/m5/exp5 LIFO, a/m5/exp6 FIFO): K1 time from the
measurement hook and a hash of V' + actions (A/B of kernel variants), plus
the converged solve's iterations and wall time."""
import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

for preset in ["a/m5/exp5", "a/m5/exp6"]:
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(3).uniform(-20.0, 20.0, n)
    P.bellman_backup_batch(m, V, 0, n)
    P.profile_enable(True)
    reps = 20
    for _ in range(reps):
        v, a = P.bellman_backup_batch(m, V, 0, n)
    ms, kl, al = P.profile_read()
    P.profile_enable(False)
    h = hashlib.sha256(v.tobytes() + a.tobytes()).hexdigest()[:16]
    t = time.perf_counter()
    r = P.run_value_iteration(m)
    w = time.perf_counter() - t
    hs = hashlib.sha256(np.asarray(r.values).tobytes()).hexdigest()[:16]
    print(f"{preset} K1 {ms / reps * 1e3:.1f} us/sweep hash {h} | solve {r.iterations} it {w:.4f} s hash {hs}")
