"""Best-of-3 wall time of the headline solves through run_value_iteration
(PVI_LOOP_TRACE=1 adds the setup / loop / extraction split):
python tools/solve_wall.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

for preset, algo in (("b/m3/exp1", "factored"), ("c/m5/exp1", "factored"), ("a/m5/exp5", "factored")):
    m = P.make_preset(preset).set_algorithm(algo)
    P.run_value_iteration(m, P.ViConfig(fixed_iterations=2))
    rs = [P.run_value_iteration(m, P.ViConfig()) for _ in range(3)]
    b = min(rs, key=lambda r: r.wall_seconds)
    print(f"{preset} {algo} it={b.iterations} wall={b.wall_seconds * 1e3:.2f} ms "
          f"kernels={b.sweep_seconds * 1e3:.2f} ms", flush=True)
