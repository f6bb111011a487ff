"""Rollout-kernel timing: simopt (config 5, b/m2/exp1 GA) and one 50-candidate
batch per scenario.  python tools/sim_ab.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

best = None
for _ in range(3):
    so = P.simopt(P.make_preset("b/m2/exp1"), rollouts_per_candidate=4096, base_seed=42, seed=1)
    best = so.device_seconds if best is None else min(best, so.device_seconds)
print(f"simopt b/m2/exp1: {len(so.log)} candidates, device {best * 1e3:.2f} ms, "
      f"{len(so.log) * 4096 * 465 / best:.3e} rollout-days/s, best {so.best}", flush=True)
cfg = P.RolloutConfig(n_rollouts=4096, base_seed=42)
for preset, params in [("a/m5/exp5", lambda i: [i % 11]), ("b/m2/exp1", lambda i: [i % 21, (i * 7) % 21]),
                       ("c/m3/exp1", lambda i: [(i + k) % 10 for k in range(7)] + [(i + k) % 10 + 10 for k in range(7)])]:
    m = P.make_preset(preset)
    pols = [P.make_heuristic_policy(m, params(i)) for i in range(50)]
    P.evaluate_policies(m, pols, cfg)
    t = time.perf_counter()
    for _ in range(3):
        P.evaluate_policies(m, pols, cfg)
    dt = (time.perf_counter() - t) / 3
    print(f"{preset}: 50 x 4096 rollouts {dt * 1e3:.2f} ms wall, {50 * 4096 * 465 / dt:.3e} rollout-days/s", flush=True)
