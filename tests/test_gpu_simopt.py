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
