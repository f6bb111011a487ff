"""Per-shard sweep time of the factored b/m3/exp1 sweep (what each rank of a
sharded run spends per sweep): contiguous x_3-pair shards (pvi_partition)
and unit shards of (pair, x_b column range) blocks (pvi_unit_partition)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("b/m3/exp1").set_algorithm("factored")
n = m.state_count()
v = torch.as_tensor(m.initial_values(), device="cuda")
w = torch.empty_like(v)
st = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def t_range(lo, hi):
    return timed(lambda: P.sweep_device(m, "f64", m.discount(), v.data_ptr(), w.data_ptr(), None, lo, hi,
                                        stream_ptr=st))


def t_units(ul, uh):
    return timed(lambda: P.sweep_device_units(m, m.discount(), v.data_ptr(), w.data_ptr(), ul, uh, stream_ptr=st))


full = t_range(0, n)
print(f"full sweep {full:.3f} ms")
for parts in (2, 4, 8):
    b = [int(x) for x in m.partition(parts)]
    ts = [t_range(b[r], b[r + 1]) for r in range(parts)]
    print(f"{parts} pair shards: " + " ".join(f"{t:.3f}" for t in ts) +
          f"  max {max(ts):.3f} ms, efficiency {full / parts / max(ts):.2f}")
    u = [int(x) for x in m.unit_partition(parts)]
    tu = [t_units(u[r], u[r + 1]) for r in range(parts)]
    print(f"{parts} unit shards: " + " ".join(f"{t:.3f}" for t in tu) +
          f"  max {max(tu):.3f} ms, efficiency {full / parts / max(tu):.2f}")
