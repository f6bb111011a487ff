"""One simopt-sized batch of rollouts (50 heuristic candidates x 4096
rollouts x 465 days on b/m2/exp1), twice -- for ncu captures of k_rollouts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("b/m2/exp1")
pols = [P.make_heuristic_policy(m, [a, b]) for a in range(5, 15) for b in range(8, 13)]
for _ in range(2):
    evs, _ = P.evaluate_policies(m, pols, P.RolloutConfig(n_rollouts=4096, base_seed=42))
print(len(evs), evs[0].ret.mean)
