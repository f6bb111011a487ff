"""GPU parity of the simulation path (K5): Philox streams, samplers,
sample_step for A/B/C, heuristic and VI-table policies, KPI accumulation
and the index-order reduction — per-rollout summaries BIT-IDENTICAL to the
reference's rollout() (sim.hpp:68-124) for a fixed seed."""
import os

import numpy as np
import pytest

from oracle import cport

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
SIM_KEYS = sorted({k.rsplit("|", 1)[0] for k in GOLD.files if k.startswith("sim|")})


def test_philox_known_answers(pvi):
    # Random123 KATs and reference RolloutRng streams
    np.testing.assert_array_equal(pvi.philox_block([0] * 4, [0] * 2), GOLD["philox|zero"])
    np.testing.assert_array_equal(pvi.philox_block([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2),
                                  GOLD["philox|ones"])
    np.testing.assert_array_equal(
        pvi.philox_block([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0]),
        GOLD["philox|pi"])
    np.testing.assert_array_equal(pvi.rollout_draws(42, 0, 0, 8), GOLD["draws|42|0|0"])
    np.testing.assert_array_equal(pvi.rollout_draws(99, 17, 364, 8), GOLD["draws|99|17|364"])
    assert [hex(x) for x in pvi.rollout_draws(42, 0, 0, 3)] == \
        ["0xd9cc07cd21677652", "0x83720ecdd211d3b4", "0xc3ad473a2d59bd1a"]


@pytest.mark.parametrize("key", SIM_KEYS)
def test_heuristic_rollouts_bitwise(pvi, key):
    _, preset, params = key.split("|")
    params = [int(x) for x in params.split(",")]
    m = pvi.make_preset(preset)
    cfg = pvi.RolloutConfig(n_rollouts=512, base_seed=42)
    (ev,), summ = pvi.evaluate_policies(m, [pvi.make_heuristic_policy(m, params)], cfg,
                                        per_rollout=True)
    np.testing.assert_array_equal(summ[0], GOLD[key + "|rollouts"])
    want = GOLD[key + "|eval"]
    got = [ev.ret.mean, ev.ret.sd, ev.service_pct[0].mean, ev.service_pct[0].sd,
           ev.service_pct[1].mean, ev.service_pct[1].sd, ev.wastage_pct[0].mean,
           ev.wastage_pct[0].sd, ev.wastage_pct[1].mean, ev.wastage_pct[1].sd,
           ev.holding_mean[0].mean, ev.holding_mean[0].sd, ev.holding_mean[1].mean,
           ev.holding_mean[1].sd]
    np.testing.assert_array_equal(np.array(got), want)


def test_vi_policy_rollouts_bitwise(pvi):
    m = pvi.make_preset("a/m2/exp1")
    res = pvi.run_value_iteration(m)
    cfg = pvi.RolloutConfig(n_rollouts=2000, base_seed=42)
    (ev,), summ = pvi.evaluate_policies(m, [pvi.make_vi_policy(m, res.policy)], cfg, per_rollout=True)
    np.testing.assert_array_equal(summ[0], GOLD["simvi|a/m2/exp1|rollouts"])
    # mean -1553.2311981713071, sd 62.308153888420009
    assert (ev.ret.mean, ev.ret.sd) == (-1553.2311981713071, 62.308153888420009)
    mb = pvi.make_preset("b/m2/exp1")
    pol = GOLD["simvi|b/m2/exp1|policy"]
    (_,), sb = pvi.evaluate_policies(mb, [pvi.make_vi_policy(mb, pol)],
                                     pvi.RolloutConfig(n_rollouts=1000, base_seed=42), per_rollout=True)
    np.testing.assert_array_equal(sb[0], GOLD["simvi|b/m2/exp1|rollouts"])


def test_batch_equals_separate_evaluations(pvi):
    """Common random numbers: evaluating candidates in one batch is
    bit-identical to evaluating them one at a time (simopt.cpp:31-34)."""
    m = pvi.make_preset("c/m3/exp2")
    cands = [[9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8],
             [5, 5, 5, 5, 5, 5, 5, 12, 12, 12, 12, 12, 12, 12],
             [0] * 14]
    cfg = pvi.RolloutConfig(n_rollouts=300, base_seed=7)
    evs, summ = pvi.evaluate_policies(m, [pvi.make_heuristic_policy(m, c) for c in cands], cfg,
                                      per_rollout=True)
    for i, c in enumerate(cands):
        (e1,), s1 = pvi.evaluate_policies(m, [pvi.make_heuristic_policy(m, c)], cfg, per_rollout=True)
        np.testing.assert_array_equal(s1[0], summ[i])
        np.testing.assert_array_equal(s1[0], cport.eval_heuristic("c/m3/exp2", c, 300, seed=7))
        assert e1.ret.mean == evs[i].ret.mean


def test_zero_horizon_conventions(pvi):
    # test_sim.cpp:81-91
    m = pvi.make_preset("a/m2/exp1")
    cfg = pvi.RolloutConfig(n_rollouts=3, horizon_days=0, warmup_days=3, base_seed=0)
    (ev,), s = pvi.evaluate_policies(m, [pvi.make_heuristic_policy(m, [2])], cfg, per_rollout=True)
    assert (s[0, :, 0] == 0.0).all() and (s[0, :, 1] == 100.0).all()
    assert (s[0, :, 3] == 0.0).all() and (s[0, :, 5] == 0.0).all()


def test_single_rollout_sd_zero(pvi):
    m = pvi.make_preset("a/m2/exp1")
    ev = pvi.evaluate_policy(m, pvi.make_heuristic_policy(m, [1]), pvi.RolloutConfig(n_rollouts=1))
    assert ev.ret.sd == 0.0


def test_never_ordering_matches_analytic_return(pvi):
    # test_sim.cpp:129-145 (A with S = 0: service 0, return -C_s E[D] annuity)
    m = pvi.make_preset("a/m2/exp1")
    ev = pvi.evaluate_policy(m, pvi.make_heuristic_policy(m, [0]),
                             pvi.RolloutConfig(n_rollouts=2000, base_seed=5))
    assert ev.service_pct[0].mean == 0.0 and ev.wastage_pct[0].mean == 0.0
    expected = -5.0 * 4.0 * (1.0 - 0.99 ** 365) / 0.01
    assert abs(ev.ret.mean - expected) <= 4.0 * ev.ret.sd / np.sqrt(2000)


def test_out_of_range_action_is_contract_violation(pvi):
    # test_sim.cpp:173-184: a VI table with an order above the cap
    m = pvi.make_preset("a/m2/exp1")
    table = np.full(121, 11, np.uint32)
    with pytest.raises(pvi.ContractViolation) as e:
        pvi.evaluate_policy(m, pvi.make_vi_policy(m, table), pvi.RolloutConfig(n_rollouts=2))
    assert "state" in str(e.value)
