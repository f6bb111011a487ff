"""Per-shard sweep time of the factored c/m5 sweeps on weekday shards
(pvi_partition: whole weekdays; launch_c_factored builds only the shard's
weekday tables): what each rank of a sharded run spends per sweep, and the
compute efficiency full / (parts x slowest shard)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for preset in ["c/m5/exp1", "c/m5/exp2"]:
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    v = torch.rand(n, dtype=torch.float64, device="cuda")
    w = torch.empty_like(v)
    st = torch.cuda.current_stream().cuda_stream
    hist = [v] * 7
    def sweep(lo, hi):
        return timed(lambda: P.sweep_device(m, "f64", m.discount(), v.data_ptr(), w.data_ptr(), None, lo, hi,
                                            "periodic_span", [h.data_ptr() for h in hist], None, st))
    full = sweep(0, n)
    print(f"{preset}: full sweep {full:.3f} ms", flush=True)
    for parts in [2, 4, 7, 8]:
        b = [int(x) for x in m.partition(parts)]
        ts = [sweep(b[r], b[r + 1]) if b[r + 1] > b[r] else 0.0 for r in range(parts)]
        print(f"  {parts} shards: max {max(ts):.3f} ms, efficiency {full / (parts * max(ts)):.2f}, "
              f"shards {[round(t, 3) for t in ts]}", flush=True)
