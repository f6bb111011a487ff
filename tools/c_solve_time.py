"""Wall / sweep time of the C factored solves (one line per preset):
python tools/c_solve_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

for preset in ("c/m5/exp1", "c/m5/exp2"):
    m = P.make_preset(preset).set_algorithm("factored")
    P.run_value_iteration(m, P.ViConfig(fixed_iterations=2))
    best = min((P.run_value_iteration(m, P.ViConfig()) for _ in range(3)), key=lambda r: r.wall_seconds)
    print(f"{preset} it={best.iterations} wall={best.wall_seconds * 1e3:.2f} ms "
          f"per_sweep={best.sweep_seconds / best.sweeps * 1e3:.3f} ms", flush=True)
