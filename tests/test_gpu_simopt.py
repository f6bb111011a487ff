"""Simulation optimisation (config 5): the reference's grid search / GA with
every generation's fresh candidates scored in one batched device launch.
Because the device rollouts are bit-identical and the host search is the
reference's algorithm on the same libstdc++ <random>, the whole search log
(candidate order, generations, mean and sd of every candidate) must equal
the reference's cmd_simopt run (tests/golden/simopt_golden.npz)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "simopt_golden.npz"))


@pytest.mark.parametrize("preset", ["a/m2/exp1", "b/m2/exp1", "c/m3/exp1"])
def test_simopt_trajectory_bitwise(pvi, preset):
    m = pvi.make_preset(preset)
    r = pvi.simopt(m, rollouts_per_candidate=4096, base_seed=42, seed=1)
    gens, n = G[f"simopt|{preset}|meta"]
    assert r.best == list(G[f"simopt|{preset}|best"])
    assert (r.best_mean, r.best_sd) == tuple(G[f"simopt|{preset}|score"])
    assert r.generations == gens and len(r.log) == n
    vals = np.array([e[1] for e in r.log])
    scores = np.array([[e[0], e[2], e[3]] for e in r.log], dtype=np.float64)
    np.testing.assert_array_equal(vals, G[f"simopt|{preset}|log_values"])
    np.testing.assert_array_equal(scores, G[f"simopt|{preset}|log_scores"])


def test_simopt_published_parameters(pvi):
    # PAPER Table 8 / Table 12: A base stock S = 5; B (S_a, S_b) = (13, 12)
    assert pvi.simopt(pvi.make_preset("a/m2/exp1"), rollouts_per_candidate=4096).best == [5]
    assert pvi.simopt(pvi.make_preset("b/m2/exp1"), rollouts_per_candidate=4096).best == [13, 12]


def test_simopt_exhaustive_grid(pvi):
    # GPU-only extra mode: all 21 x 21 (S_a, S_b) in one batch.
    # Common random numbers: every candidate the reference's GA scored has the
    # same (mean, sd) bit for bit, and the grid's best is the global optimum
    # of the GA's ordering (higher mean, then the smaller vector).
    m = pvi.make_preset("b/m2/exp1")
    r = pvi.simopt(m, sampler="exhaustive", rollouts_per_candidate=4096, base_seed=42)
    assert len(r.log) == 441 and r.generations == 1
    vals = [tuple(e[1]) for e in r.log]
    assert vals == sorted(vals) and len(set(vals)) == 441
    score = {tuple(e[1]): (e[2], e[3]) for e in r.log}
    for v, (_, mean, sd) in zip(G["simopt|b/m2/exp1|log_values"], G["simopt|b/m2/exp1|log_scores"]):
        assert score[tuple(int(x) for x in v)] == (mean, sd)
    top = max(r.log, key=lambda e: (e[2], [-x for x in e[1]]))
    assert r.best == list(top[1]) and r.best_mean == top[2]
    assert r.best_mean >= G["simopt|b/m2/exp1|score"][0]
    with pytest.raises(pvi.ParameterError):  # 21^14 candidates
        pvi.simopt(pvi.make_preset("c/m3/exp1"), sampler="exhaustive", rollouts_per_candidate=16)
