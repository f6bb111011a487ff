"""A/B of the solve loop control and the L2 window on one GPU:
python tools/loop_ab.py  -> one line per (preset, algorithm, loop, l2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

CASES = [("a/m2/exp1", "exact"), ("a/m5/exp5", "factored"), ("a/m5/exp6", "factored"),
         ("a/m5/exp5", "exact"), ("b/m3/exp1", "factored"), ("b/m2/exp1", "exact"),
         ("c/m5/exp1", "factored"), ("c/m5/exp2", "factored"), ("c/m3/exp1", "exact")]
for preset, algo in CASES:
    m = P.make_preset(preset).set_algorithm(algo)
    P.run_value_iteration(m, P.ViConfig(fixed_iterations=2))  # warm tables / scratch
    for loop in ("host", "graph"):
        for l2 in (False, True):
            best = None
            for _ in range(2):
                r = P.run_value_iteration(m, P.ViConfig(loop=loop, l2_persist=l2))
                if best is None or r.wall_seconds < best.wall_seconds:
                    best = r
            print(f"{preset:10s} {algo:8s} loop={loop:5s} l2={int(l2)} it={best.iterations:5d} "
                  f"wall={best.wall_seconds * 1e3:9.2f} ms  sweep={best.sweep_seconds * 1e3:9.2f} ms "
                  f"per_sweep={best.wall_seconds / max(best.iterations, 1) * 1e6:8.1f} us "
                  f"graph_sweeps={best.graph_sweeps} l2_bytes={best.l2_window_bytes} "
                  f"hit={best.l2_hit_ratio:.3f}", flush=True)
