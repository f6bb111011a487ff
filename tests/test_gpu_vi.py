"""GPU parity of the value-iteration path (K1 backup, K2 fused convergence
reduction, K3 policy extraction, K4 initial value) against the reference.

The device kernels reproduce the reference's per-term arithmetic and
summation order with no FMA contraction, so in f64 AND f32 the value
vectors, iteration counts and policies must be BIT-IDENTICAL to the
reference's run_value_iteration (vi.hpp:295) — stronger than the north
star's 1e-9 / +-1 iteration / near-tie bar.  Expected values come from
tests/golden/reference_golden.npz (reference outputs) and the C oracle.
"""
import hashlib
import os

import numpy as np
import pytest

from oracle import cport

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
SOLVE_KEYS = sorted({k.rsplit("|", 1)[0] for k in GOLD.files if k.startswith("solve|")})


@pytest.mark.parametrize("key", SOLVE_KEYS)
def test_solve_bitwise_vs_reference(pvi, key):
    _, preset, prec = key.split("|")
    res = pvi.run_value_iteration(pvi.make_preset(preset), pvi.ViConfig(precision=prec))
    it, conv = GOLD[key + "|meta"]
    assert res.iterations == it and res.converged == bool(conv)
    np.testing.assert_array_equal(res.values, GOLD[key + "|values"])
    np.testing.assert_array_equal(res.policy, GOLD[key + "|policy"])


@pytest.mark.parametrize("preset,k", [("b/m2/p1", 100), ("b/m2/p4", 100), ("b/m3/exp4", 2)])
def test_fixed_iterations_bitwise(pvi, preset, k):
    res = pvi.run_value_iteration(pvi.make_preset(preset), pvi.ViConfig(fixed_iterations=k))
    assert res.iterations == k and res.converged
    key = f"fixed|{preset}|{k}"
    if key + "|values" in GOLD.files:
        np.testing.assert_array_equal(res.values, GOLD[key + "|values"])
        np.testing.assert_array_equal(res.policy, GOLD[key + "|policy"])
    else:
        assert hashlib.sha256(res.values.tobytes()).digest() == GOLD[key + "|values_sha256"].tobytes()
        assert hashlib.sha256(res.policy.tobytes()).digest() == GOLD[key + "|policy_sha256"].tobytes()


def test_headline_sweep_b_m3_exp1(pvi):
    """One f64 sweep of the 16,777,216-state instance from V0 (SURVEY App. B,
    reference flags): V1[0] = 3.43438095058583, V1[-1] = 19.999999999999908;
    a slice of the sweep is bit-identical to the C oracle."""
    m = pvi.make_preset("b/m3/exp1")
    res = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=1))
    assert repr(float(res.values[0])) == "3.43438095058583"
    assert repr(float(res.values[-1])) == "19.999999999999908"
    v0 = m.initial_values()
    lo, hi = 8388608 + 4096 * 3, 8388608 + 4096 * 3 + 640
    wv, wa = cport.backup_range("b/m3/exp1", v0, lo, hi)
    np.testing.assert_array_equal(res.values[lo:hi], wv)
    gv, ga = pvi.bellman_backup_batch(m, v0, lo, hi)
    np.testing.assert_array_equal(gv, wv)
    np.testing.assert_array_equal(ga, wa)


@pytest.mark.parametrize("preset", ["b/m3/exp1", "b/m3/exp4", "c/m5/exp1", "c/m5/exp2",
                                    "a/m5/exp5", "a/m5/exp8"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_q_rows_bitwise(pvi, preset, prec):
    m = pvi.make_preset(preset)
    V = np.random.default_rng(7).uniform(-5.0, 5.0, m.state_count())
    states = GOLD[f"qrow|{preset}|states"]
    got = np.stack([pvi.q_rows(m, V, int(s), int(s) + 1, precision=prec)[0] for s in states])
    if prec == "f64":
        np.testing.assert_array_equal(got, GOLD[f"qrow|{preset}|q"])
    else:
        want = np.stack([cport.q_row(preset, int(s), V, f32=True) for s in states])
        np.testing.assert_array_equal(got.astype(np.float64), want)


@pytest.mark.parametrize("preset,lo,count", [("c/m5/exp1", 680000, 64), ("c/m3/exp2", 0, 3087),
                                             ("a/m5/exp5", 1000000, 4096),
                                             ("b/m2/exp2", 0, 11025), ("b/m3/exp2", 5000000, 512)])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_backup_slices_bitwise(pvi, preset, lo, count, prec):
    m = pvi.make_preset(preset)
    V = np.random.default_rng(11).uniform(-100.0, 100.0, m.state_count())
    if prec == "f32":
        V = V.astype(np.float32).astype(np.float64)
    gv, ga = pvi.bellman_backup_batch(m, V, lo, lo + count, precision=prec)
    wv, wa = cport.backup_range(preset, V, lo, lo + count, f32=prec == "f32")
    np.testing.assert_array_equal(gv.astype(np.float64), wv)
    np.testing.assert_array_equal(ga, wa)


def test_sub_range_invariance(pvi):
    """Batch-size invariance (test_vi.cpp:177-195): any split of the state
    range gives the same bits as one sweep."""
    m = pvi.make_preset("b/m2/p4")
    V = np.random.default_rng(5).uniform(-10, 10, m.state_count())
    full_v, full_a = pvi.bellman_backup_batch(m, V, 0, m.state_count())
    cuts = [0, 1, 7, 200, 201, 9000, 20000, m.state_count()]
    parts = [pvi.bellman_backup_batch(m, V, a, b) for a, b in zip(cuts, cuts[1:])]
    np.testing.assert_array_equal(np.concatenate([p[0] for p in parts]), full_v)
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), full_a)


def test_initial_values_bitwise(pvi):
    np.testing.assert_array_equal(pvi.make_preset("b/m2/exp1").initial_values(), GOLD["v0|b/m2/exp1"])
    v0 = pvi.make_preset("b/m3/exp4").initial_values()
    idx = GOLD["v0sample|b/m3/exp4|states"]
    np.testing.assert_array_equal(v0[idx], GOLD["v0sample|b/m3/exp4|values"])


# --- explicit-table MDPs (tests/support/tabular_mdp.hpp, test_vi.cpp) ------

TAB_KEYS = sorted({k.rsplit("|", 1)[0] for k in GOLD.files if k.startswith("tab|")})


def _tab(pvi, key, prefix="tab"):
    if prefix == "tab":
        _, ns, na, no, g, _seed = key.split("|")
        ns, na, no, g = int(ns), int(na), int(no), float(g)
    else:
        ns, na, no, _seed = (int(x) for x in GOLD[key + "|dims"])
        g = 0.9
    return pvi.TabularMdp(ns, na, no, g, GOLD[key + "|next"], GOLD[key + "|reward"],
                          GOLD[key + "|prob"]), ns


@pytest.mark.parametrize("key", TAB_KEYS)
def test_tabular_solve_bitwise(pvi, key):
    m, ns = _tab(pvi, key)
    res = pvi.run_value_iteration(m, pvi.ViConfig(epsilon=1e-12))
    it, conv = GOLD[key + "|meta"]
    assert res.iterations == it and res.converged == bool(conv)
    np.testing.assert_array_equal(res.values, GOLD[key + "|values"])
    np.testing.assert_array_equal(res.policy, GOLD[key + "|policy"])


@pytest.mark.parametrize("t", range(10))
def test_tabular_brute_force_policy(pvi, t):
    """test_vi.cpp:74-91: VI policy equals brute-force enumeration."""
    key = f"brute|{t}"
    m, ns = _tab(pvi, key, "brute")
    res = pvi.run_value_iteration(m, pvi.ViConfig(epsilon=1e-12))
    np.testing.assert_array_equal(res.policy, GOLD[key + "|brute_policy"])
    np.testing.assert_allclose(res.values, GOLD[key + "|brute_values"], rtol=1e-6)
    np.testing.assert_array_equal(res.values, GOLD[key + "|values"])


def test_single_state_backup_and_fixed_point(pvi):
    # test_vi.cpp:31-48
    m = pvi.TabularMdp(1, 1, 1, 0.5, [0], [1.0], [1.0])
    v, a = pvi.bellman_backup_batch(m, np.zeros(1), 0, 1, gamma=0.5)
    assert v[0] == 1.0 and a[0] == 0
    res = pvi.run_value_iteration(m, pvi.ViConfig(epsilon=1e-10))
    assert res.converged and abs(res.values[0] - 2.0) < 1e-8


def test_argmax_ties_break_to_smallest_action(pvi):
    # test_vi.cpp:93-104
    m = pvi.TabularMdp(1, 3, 1, 0.0, [0, 0, 0], [1.0, 1.0, 1.0], [1.0, 1.0, 1.0])
    _, a = pvi.bellman_backup_batch(m, np.zeros(1), 0, 1, gamma=0.0)
    assert a[0] == 0


def test_numeric_divergence_reports_iteration(pvi):
    # test_vi.cpp:225-240
    m = pvi.TabularMdp(2, 1, 1, 1.0, [0, 1], [1e308, 1e308], [1.0, 1.0])
    with pytest.raises(pvi.NumericDivergence) as e:
        pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=10))
    assert e.value.iteration == 2
    assert "state 0" in str(e.value)


def test_capacity_gate(pvi):
    # test_vi.cpp:242-252
    key = "tab|64|2|2|0.9|3"
    m, _ = _tab(pvi, key)
    with pytest.raises(pvi.CapacityError) as e:
        pvi.run_value_iteration(m, pvi.ViConfig(max_states=63))
    assert e.value.required_count == 64


def test_convergence_tests_truth_tables(pvi):
    # test_vi.cpp:106-147, evaluated by the device reduction kernel
    m = pvi.TabularMdp(2, 1, 1, 0.9, [0, 1], [0.0, 0.0], [1.0, 1.0])
    same = [np.array([1.0, 2.0]), np.array([1.0, 2.0])]
    assert pvi.check_convergence(m, "value_span", same, 0.9, 1e-12, 3)
    assert pvi.check_convergence(m, "change_span", same, 0.9, 1e-12, 3)
    shifted = [np.array([1.0, 2.0]), np.array([2.5, 3.5])]
    assert not pvi.check_convergence(m, "value_span", shifted, 0.9, 1e-4, 3)
    assert pvi.check_convergence(m, "change_span", shifted, 0.9, 1e-4, 3)
    with pytest.raises(pvi.ContractViolation):
        pvi.check_convergence(m, "value_span", [np.array([1.0, 2.0])], 0.9, 1e-4, 3)
    with pytest.raises(pvi.ContractViolation):
        pvi.check_convergence(m, "periodic_span", shifted, 0.9, 1e-4, 9)
    m3 = pvi.TabularMdp(3, 1, 1, 0.95, [0, 1, 2], [0.0] * 3, [1.0] * 3)

    def hist(base, slope):
        return [np.array([b + k * s for b, s in zip(base, slope)]) for k in range(8)]
    uniform = hist([5.0, -2.0, 0.5], [1.5, 1.5, 1.5])
    assert pvi.check_convergence(m3, "periodic_span", uniform, 0.95, 1e-4, 12)
    assert not pvi.check_convergence(m3, "periodic_span", uniform, 0.95, 1e-4, 6)
    skewed = hist([5.0, -2.0, 0.5], [1.5, 1.6, 1.5])
    assert not pvi.check_convergence(m3, "periodic_span", skewed, 0.95, 1e-4, 12)


def test_resume_reproduces_uninterrupted_run(pvi, tmp_path):
    # test_vi.cpp:197-223 and :277-300, through PVI1 checkpoints
    key = "tab|15|3|4|0.9|808"
    m, _ = _tab(pvi, key)
    full = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=10))
    path = str(tmp_path / "r.ckpt")
    pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=6, checkpoint_every=6,
                                            checkpoint_path=path))
    ck = pvi.load_checkpoint(path, m.fingerprint())
    assert ck.iteration == 6
    resumed = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=10), resume=ck)
    assert resumed.iterations == 10
    np.testing.assert_array_equal(resumed.values, full.values)
    np.testing.assert_array_equal(resumed.policy, full.policy)
    # convergence-tested resume lands on the same fixed point
    m2, _ = _tab(pvi, "tab|12|3|4|0.85|2712")
    unint = pvi.run_value_iteration(m2, pvi.ViConfig(epsilon=1e-10))
    part = pvi.run_value_iteration(m2, pvi.ViConfig(epsilon=1e-10, max_iterations=5,
                                                    checkpoint_every=5, checkpoint_path=path))
    assert not part.converged
    res = pvi.run_value_iteration(m2, pvi.ViConfig(epsilon=1e-10),
                                  resume=pvi.load_checkpoint(path, m2.fingerprint()))
    assert res.converged and res.iterations == unint.iterations
    np.testing.assert_array_equal(res.values, unint.values)


def test_resume_refuses_foreign_fingerprint(pvi, tmp_path):
    m = pvi.make_preset("a/m2/exp1")
    ck = pvi.Checkpoint(np.zeros(121), 3, pvi.sha256(b"other"))
    with pytest.raises(pvi.FingerprintMismatch):
        pvi.run_value_iteration(m, resume=ck)


def test_preset_checkpoints_each_sweep(pvi, tmp_path):
    """B/C presets checkpoint every sweep (presets.cpp:111,122); the final
    checkpoint holds the converged V widened to f64."""
    m = pvi.make_preset("b/m2/exp1")
    path = str(tmp_path / "b.ckpt")
    res = pvi.run_value_iteration(m, pvi.ViConfig(checkpoint_every=1, checkpoint_path=path))
    ck = pvi.load_checkpoint(path, m.fingerprint())
    assert ck.iteration == res.iterations == 12
    np.testing.assert_array_equal(ck.values, res.values)


@pytest.mark.parametrize("preset", ["a/m2/exp1", "b/m2/exp1", "c/m3/exp1"])
def test_sharded_driver_world1_equals_solver(pvi, preset):
    """The multi-GPU driver (device sweep through pvi_vi_sweep_device + the
    reduced statistic) gives the single-GPU solver's bits at world size 1."""
    from paper_2303_10672_b200.sharded import ShardedValueIteration
    m = pvi.make_preset(preset)
    res = ShardedValueIteration(m).solve()
    key = f"solve|{preset}|f64"
    assert res.iterations == GOLD[key + "|meta"][0]
    np.testing.assert_array_equal(res.values, GOLD[key + "|values"])
    np.testing.assert_array_equal(res.policy, GOLD[key + "|policy"])


@pytest.mark.gpu
@pytest.mark.parametrize("preset,algo,prec", [("c/m5/exp1", "factored", "f64"), ("a/m5/exp5", "factored", "f64"),
                                              ("b/m2/exp1", "exact", "f64"), ("b/m3/exp1", "factored", "f32")])
def test_pageable_and_pinned_readback_identical(pvi, preset, algo, prec):
    """Result buffers in pageable memory go through the engine's pinned ring
    and host copy pool (several 8 MB chunks here), pinned ones take one
    direct copy: the same bytes either way, and the same as a range split."""
    import torch
    m = pvi.make_preset(preset).set_algorithm(algo)
    n = m.state_count()
    V = np.random.default_rng(21).uniform(-10.0, 10.0, n)
    tdt = torch.float32 if prec == "f32" else torch.float64
    v_pg, a_pg = pvi.bellman_backup_batch(m, V, 0, n, precision=prec)  # numpy: pageable
    ov = torch.empty(n, dtype=tdt).pin_memory().numpy()
    oa = torch.empty(n, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    v_pn, a_pn = pvi.bellman_backup_batch(m, V, 0, n, precision=prec, out_values=ov, out_actions=oa)
    np.testing.assert_array_equal(v_pg, v_pn)
    np.testing.assert_array_equal(a_pg, a_pn)
    half = n // 2 + 7
    v1, a1 = pvi.bellman_backup_batch(m, V, 0, half, precision=prec)
    np.testing.assert_array_equal(v1, v_pg[:half])
    np.testing.assert_array_equal(a1, a_pg[:half])
    if prec == "f32":
        return
    # the solve's read-back (pageable numpy result) equals three backups
    res = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=3))
    v = np.asarray(m.initial_values(), np.float64)
    for _ in range(3):
        v, a = pvi.bellman_backup_batch(m, v, 0, n)
    np.testing.assert_array_equal(res.values, v)
    _, pol = pvi.bellman_backup_batch(m, v, 0, n)
    np.testing.assert_array_equal(res.policy, pol)
