PVI_LOOP_TRACE=1 python - <<'P'
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2303_10672_b200 as P
m = P.make_preset("b/m3/exp1").set_algorithm("factored")
n = m.state_count()
vh = torch.as_tensor(m.initial_values()).pin_memory().numpy()
ov = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
oa = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
for i in range(4):
    t = time.perf_counter()
    P.bellman_backup_batch(m, vh, 0, n, out_values=ov, out_actions=oa)
    print("call", i, f"{1e3*(time.perf_counter()-t):.3f} ms", flush=True)
P
