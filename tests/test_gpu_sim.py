"""GPU parity of the simulation path: per-rollout summaries bit-identical to
the reference's rollout() (sim.hpp:68-124) for a fixed seed."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_philox_kat(pvi):
    # Random123 known-answer vectors.
    assert [hex(x) for x in pvi.philox_block([0, 0, 0, 0], [0, 0])] == \
        ["0x6627e8d5", "0xe169c58d", "0xbc57ac4c", "0x9b00dbd8"]
    ones = 0xFFFFFFFF
    assert [hex(x) for x in pvi.philox_block([ones] * 4, [ones] * 2)] == \
        ["0x408f276d", "0x41c83b0e", "0xa20bc7c6", "0x6d5451fd"]
    assert [hex(x) for x in pvi.rollout_draws(42, 0, 0, 3)] == \
        ["0xd9cc07cd21677652", "0x83720ecdd211d3b4", "0xc3ad473a2d59bd1a"]


@pytest.mark.parametrize("preset,params", [("a/m2/exp1", [5]), ("a/m3/exp6", [7]),
                                           ("b/m2/exp1", [13, 12]),
                                           ("c/m3/exp1", [9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8])])
def test_heuristic_rollouts_bitwise(pvi, ref, preset, params):
    m = pvi.make_preset(preset)
    cfg = pvi.RolloutConfig(n_rollouts=512, base_seed=42)
    (ev,), summ = pvi.evaluate_policies(m, [pvi.make_heuristic_policy(m, params)], cfg, per_rollout=True)
    want, want_ev = ref.eval_heuristic(preset, params, 512, seed=42)
    np.testing.assert_array_equal(summ[0], want)
    assert ev.ret.mean == want_ev[0] and ev.ret.sd == want_ev[1]


def test_vi_policy_rollouts_bitwise(pvi, ref):
    preset = "a/m2/exp1"
    m = pvi.make_preset(preset)
    res = pvi.run_value_iteration(m)
    cfg = pvi.RolloutConfig(n_rollouts=2000, base_seed=42)
    ev = pvi.evaluate_policy(m, pvi.make_vi_policy(m, res.policy), cfg)
    # mean -1553.2311981713071, sd 62.308153888420009
    assert ev.ret.mean == -1553.2311981713071
    assert ev.ret.sd == 62.308153888420009
