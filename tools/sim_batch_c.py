"""One 50-candidate x 4096-rollout batch of (s, S) heuristics on c/m3/exp1,
twice -- for ncu captures of the C rollout kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("c/m3/exp1")
pols = [P.make_heuristic_policy(m, [(i + k) % 10 for k in range(7)] + [(i + k) % 10 + 10 for k in range(7)])
        for i in range(50)]
for _ in range(2):
    evs, _ = P.evaluate_policies(m, pols, P.RolloutConfig(n_rollouts=4096, base_seed=42))
print(len(evs), evs[0].ret.mean)
