"""Converged-solve wall time of one preset, best of N solves in one process
(the first pays tables / graph instantiation):
    python tools/solve_repeat.py a/m5/exp5 [factored] [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

preset = sys.argv[1] if len(sys.argv) > 1 else "a/m5/exp5"
algo = sys.argv[2] if len(sys.argv) > 2 else "factored"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 5
m = P.make_preset(preset).set_algorithm(algo)
walls = []
for _ in range(n):
    r = P.run_value_iteration(m)
    walls.append(r.wall_seconds)
print(f"{preset} {algo}: {r.iterations} sweeps, solve wall best {min(walls):.4f} s, all "
      + " ".join(f"{w:.4f}" for w in walls))
