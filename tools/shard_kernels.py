"""One sweep of each unit shard of the factored b/m3/exp1 sweep at `parts`
ranks (default 8), for an ncu launch list: which kernel carries the
per-shard fixed cost.  Usage: ncu --metrics gpu__time_duration.sum
--clock-control none --csv python tools/shard_kernels.py [parts]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
m = P.make_preset("b/m3/exp1").set_algorithm("factored")
v = torch.as_tensor(m.initial_values(), device="cuda")
w = torch.empty_like(v)
st = torch.cuda.current_stream().cuda_stream
u = [int(x) for x in m.unit_partition(parts)]
P.sweep_device_units(m, m.discount(), v.data_ptr(), w.data_ptr(), 0, u[-1], stream_ptr=st)  # tables, scratch
torch.cuda.synchronize()
for r in range(parts):
    P.sweep_device_units(m, m.discount(), v.data_ptr(), w.data_ptr(), u[r], u[r + 1], stream_ptr=st)
    torch.cuda.synchronize()
print("units", u)
