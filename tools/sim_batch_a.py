"""One 50-candidate x 4096-rollout batch of base-stock heuristics on a/m5/exp5,
twice -- for ncu captures of the A rollout kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

m = P.make_preset("a/m5/exp5")
pols = [P.make_heuristic_policy(m, [i % 11]) for i in range(50)]
for _ in range(2):
    evs, _ = P.evaluate_policies(m, pols, P.RolloutConfig(n_rollouts=4096, base_seed=42))
print(len(evs), evs[0].ret.mean)
