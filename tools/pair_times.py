"""Per-shard sweep time of the factored b/m3/exp1 sweep for 1..8-way
partitions (what each rank of a sharded run would spend per sweep)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("b/m3/exp1").set_algorithm("factored")
n = m.state_count()
v = torch.as_tensor(m.initial_values(), device="cuda")
w = torch.empty_like(v)
st = torch.cuda.current_stream().cuda_stream


def t_shard(lo, hi, reps=5):
    for _ in range(2):
        P.sweep_device(m, "f64", m.discount(), v.data_ptr(), w.data_ptr(), None, lo, hi, stream_ptr=st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        P.sweep_device(m, "f64", m.discount(), v.data_ptr(), w.data_ptr(), None, lo, hi, stream_ptr=st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = t_shard(0, n)
print(f"full sweep {full:.3f} ms")
for parts in (2, 4, 8):
    b = [int(x) for x in m.partition(parts)]
    ts = [t_shard(b[r], b[r + 1]) for r in range(parts)]
    print(f"{parts} shards: " + " ".join(f"{t:.3f}" for t in ts) +
          f"  max {max(ts):.3f} ms, ideal {full / parts:.3f} ms, efficiency {full / parts / max(ts):.2f}")
