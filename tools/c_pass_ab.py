"""Factored-C sweeps for A/B of kernel versions: full c/m5 (and c/m3/exp2)
sweeps on a seeded V, K1 time from the measurement hook and a SHA-256 of
V' + argmax (bit-identical versions print the same hash).  Compare builds
with tools/with_lib.py.

    python tools/c_pass_ab.py
"""
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

for preset in ["c/m5/exp1", "c/m5/exp2", "c/m3/exp2"]:
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(3).uniform(-20.0, 20.0, n)
    P.bellman_backup_batch(m, V, 0, n)
    P.profile_enable(True)
    reps = 5
    for _ in range(reps):
        v, a = P.bellman_backup_batch(m, V, 0, n)
    ms, kl, al = P.profile_read()
    P.profile_enable(False)
    h = hashlib.sha256(v.tobytes() + a.tobytes()).hexdigest()[:16]
    print(f"{preset} K1 {ms / reps:.3f} ms/sweep hash {h}")
