"""Exact (reference-order) b/m3/exp1 sweep: device time of bench's alternate
step (pvi_vi_sweep_device on resident buffers), best of 3, and a hash."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "b/m3/exp1"
m = P.make_preset(preset)
n = m.state_count()
v = torch.as_tensor(m.initial_values(), device="cuda")
w = torch.empty_like(v)
st = torch.cuda.current_stream().cuda_stream
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.sweep_device(m, "f64", m.discount(), v.data_ptr(), w.data_ptr(), None, 0, n, stream_ptr=st)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
h = hashlib.sha256(w.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{preset} exact sweep {best:.1f} ms hash {h}")
