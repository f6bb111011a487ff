"""Host-buffer backup of b/m3/exp1 (bench.py's e2e leg) with the pipeline's
event trace (PVI_LOOP_TRACE=1 prints the piece timestamps to stderr).
    PVI_LOOP_TRACE=1 python tools/e2e_trace.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("b/m3/exp1").set_algorithm("factored")
n = m.state_count()
v0 = np.random.default_rng(7).uniform(-5, 5, n)
vh = torch.as_tensor(v0).pin_memory().numpy()
ov = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
oa = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
for _ in range(3):
    P.bellman_backup_batch(m, vh, 0, n, out_values=ov, out_actions=oa)
ts = []
for _ in range(int(os.environ.get("REPS", "5"))):
    t0 = time.perf_counter()
    P.bellman_backup_batch(m, vh, 0, n, out_values=ov, out_actions=oa)
    ts.append((time.perf_counter() - t0) * 1e3)
print("e2e ms:", " ".join(f"{t:.3f}" for t in ts))
