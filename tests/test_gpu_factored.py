"""The factored Scenario B sweep (algorithm = "factored") against the
reference under the north-star contract: V within 1e-9 relative (we check
1e-12), the same iteration count, and the same policy except at documented
near-ties (|Q(a_ours) - Q(a_ref)| below 1e-9 relative, checked with the
exact Q rows)."""
import hashlib
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def _near_tie_ok(pvi, preset, values, got_policy, want_policy, rel=1e-9):
    bad = np.nonzero(got_policy != want_policy)[0]
    if len(bad) == 0:
        return 0
    m = pvi.make_preset(preset)  # exact Q rows at the converged V
    for s in bad:
        q = pvi.q_rows(m, values, int(s), int(s) + 1)[0]
        a, b = int(got_policy[s]), int(want_policy[s])
        assert abs(q[a] - q[b]) <= rel * max(1.0, abs(q[b])), (s, q[a], q[b])
    return len(bad)


@pytest.mark.parametrize("preset", ["b/m2/exp1", "b/m2/exp2"])
def test_factored_solve_matches_reference(pvi, preset):
    m = pvi.make_preset(preset).set_algorithm("factored")
    res = pvi.run_value_iteration(m)
    key = f"solve|{preset}|f64"
    it, conv = GOLD[key + "|meta"]
    assert res.iterations == it and res.converged == bool(conv)
    want = GOLD[key + "|values"]
    np.testing.assert_allclose(res.values, want, rtol=1e-12, atol=0)
    _near_tie_ok(pvi, preset, res.values, res.policy, GOLD[key + "|policy"])


@pytest.mark.parametrize("preset,k", [("b/m2/p1", 100), ("b/m2/p4", 100)])
def test_factored_fixed_iterations(pvi, preset, k):
    m = pvi.make_preset(preset).set_algorithm("factored")
    res = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=k))
    key = f"fixed|{preset}|{k}"
    np.testing.assert_allclose(res.values, GOLD[key + "|values"], rtol=1e-11, atol=0)
    _near_tie_ok(pvi, preset, res.values, res.policy, GOLD[key + "|policy"])


def test_factored_b_m3_exp4_two_sweeps(pvi):
    m = pvi.make_preset("b/m3/exp4").set_algorithm("factored")
    res = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=2))
    idx = GOLD["fixed|b/m3/exp4|2|sample_states"]
    np.testing.assert_allclose(res.values[idx], GOLD["fixed|b/m3/exp4|2|sample_values"],
                               rtol=1e-12, atol=0)


def test_factored_headline_first_sweep(pvi):
    m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
    res = pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=1))
    assert abs(res.values[0] - 3.43438095058583) <= 1e-12 * 3.43438095058583
    assert abs(res.values[-1] - 19.999999999999908) <= 1e-12 * 20.0


@pytest.mark.parametrize("preset", ["b/m3/exp1", "b/m3/exp4", "b/m2/p3"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_factored_q_rows_close_to_exact(pvi, preset, prec):
    exact = pvi.make_preset(preset)
    fact = pvi.make_preset(preset).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(3).uniform(-5.0, 5.0, n)
    lo = (n // 3) // 4096 * 4096
    hi = min(n, lo + 4096)
    qe = pvi.q_rows(exact, V, lo, hi, precision=prec).astype(np.float64)
    qf = pvi.q_rows(fact, V, lo, hi, precision=prec).astype(np.float64)
    tol = 1e-12 if prec == "f64" else 2e-6
    np.testing.assert_allclose(qf, qe, rtol=tol, atol=tol)


# --- Scenario C: demand summed per post-delivery profile first ------------

@pytest.mark.parametrize("preset", ["c/m3/exp1", "c/m3/exp2"])
def test_factored_c_solve_matches_reference(pvi, preset):
    m = pvi.make_preset(preset).set_algorithm("factored")
    res = pvi.run_value_iteration(m)
    key = f"solve|{preset}|f64"
    it, conv = GOLD[key + "|meta"]
    assert res.iterations == it and res.converged == bool(conv)
    np.testing.assert_allclose(res.values, GOLD[key + "|values"], rtol=1e-12, atol=0)
    _near_tie_ok(pvi, preset, res.values, res.policy, GOLD[key + "|policy"])


@pytest.mark.parametrize("preset", ["c/m5/exp1", "c/m5/exp2", "c/m3/exp2"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_factored_c_q_rows_close_to_exact(pvi, preset, prec):
    exact = pvi.make_preset(preset)
    fact = pvi.make_preset(preset).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(9).uniform(-50.0, 50.0, n)
    lo = n // 2
    hi = min(n, lo + 512)
    qe = pvi.q_rows(exact, V, lo, hi, precision=prec).astype(np.float64)
    qf = pvi.q_rows(fact, V, lo, hi, precision=prec).astype(np.float64)
    tol = 1e-12 if prec == "f64" else 2e-6
    np.testing.assert_allclose(qf, qe, rtol=tol, atol=tol * 100)
    golden = GOLD.get(f"qrow|{preset}|q") if f"qrow|{preset}|q" in GOLD.files else None
    if golden is not None and prec == "f64":
        V7 = np.random.default_rng(7).uniform(-5.0, 5.0, n)
        for i, s in enumerate(GOLD[f"qrow|{preset}|states"]):
            q = pvi.q_rows(fact, V7, int(s), int(s) + 1)[0]
            np.testing.assert_allclose(q, golden[i], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("preset,parts", [("b/m3/exp1", 8), ("b/m3/exp4", 3), ("c/m5/exp1", 4),
                                          ("b/m2/p4", 5)])
def test_factored_shards_equal_full_sweep(pvi, preset, parts):
    """What each rank of the sharded driver computes (its cost-weighted,
    group-aligned [lo, hi) slice) is bit-identical to that slice of a
    single full sweep."""
    m = pvi.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(5).uniform(-20.0, 20.0, n)
    full_v, full_a = pvi.bellman_backup_batch(m, V, 0, n)
    bounds = [int(b) for b in m.partition(parts)]
    assert bounds[0] == 0 and bounds[-1] == n
    for lo, hi in zip(bounds, bounds[1:]):
        v, a = pvi.bellman_backup_batch(m, V, lo, hi)
        np.testing.assert_array_equal(v, full_v[lo:hi])
        np.testing.assert_array_equal(a, full_a[lo:hi])
    # an arbitrary unaligned range as well
    lo, hi = n // 3 + 17, n // 3 + 17 + 5000
    v, a = pvi.bellman_backup_batch(m, V, lo, hi)
    np.testing.assert_array_equal(v, full_v[lo:hi])


@pytest.mark.parametrize("preset", ["c/m5/exp1", "c/m5/exp2"])
def test_factored_c_full_sweep_close_to_exact(pvi, preset):
    """Whole-space backup: c/m5/exp1 has an exogenous receipt law (scalar
    anti-diagonal passes k_c_bin_diag + the fused k_c_bin_diag_qf); exp2 is
    endogenous (the DMMA passes k_c_bin_wide_mma + the fused pass-2/Q
    k_c_bin_diag_q).  Both agree with the exact (reference-order) sweep to
    rounding."""
    exact = pvi.make_preset(preset)
    fact = pvi.make_preset(preset).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(11).uniform(-30.0, 30.0, n)
    ve, ae = pvi.bellman_backup_batch(exact, V, 0, n)
    vf, af = pvi.bellman_backup_batch(fact, V, 0, n)
    np.testing.assert_allclose(vf, ve, rtol=1e-12, atol=1e-10)
    bad = np.nonzero(af != ae)[0]
    assert len(bad) <= n // 10000
    for s in bad:
        q = pvi.q_rows(exact, V, int(s), int(s) + 1)[0]
        assert abs(q[af[s]] - q[ae[s]]) <= 1e-9 * max(1.0, abs(q[ae[s]]))


@pytest.mark.parametrize("preset", ["b/m3/exp1", "b/m3/exp4"])
def test_factored_b_full_sweep_close_to_exact(pvi, preset):
    """Whole-space backup against the exact (reference-order) sweep: every
    x_a digit pattern goes through the diagonal stage-2 kernel
    (k_b_fact_qw4 on b/m3/exp1)."""
    exact = pvi.make_preset(preset)
    fact = pvi.make_preset(preset).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(13).uniform(-8.0, 8.0, n)
    ve, ae = pvi.bellman_backup_batch(exact, V, 0, n)
    vf, af = pvi.bellman_backup_batch(fact, V, 0, n)
    np.testing.assert_allclose(vf, ve, rtol=1e-12, atol=1e-11)
    bad = np.nonzero(af != ae)[0]
    assert len(bad) <= n // 10000
    for s in bad:
        q = pvi.q_rows(exact, V, int(s), int(s) + 1)[0]
        assert abs(q[af[s]] - q[ae[s]]) <= 1e-9 * max(1.0, abs(q[ae[s]]))
    # scattered single-state Q rows (every order pair)
    for s in np.random.default_rng(14).integers(0, n, 16):
        np.testing.assert_allclose(pvi.q_rows(fact, V, int(s), int(s) + 1),
                                   pvi.q_rows(exact, V, int(s), int(s) + 1), rtol=1e-12, atol=1e-11)


# --- Scenario A: demand values that leave the same carried stock merged ---

@pytest.mark.parametrize("preset", ["a/m2/exp1", "a/m2/exp2", "a/m2/exp6", "a/m3/exp5"])
def test_factored_a_solve_matches_reference(pvi, preset):
    """LIFO (exp1, exp5) and FIFO (exp2, exp6), lead times 1 and 2: values
    within 1e-9 of the reference (value-span solves run ~1,000 sweeps, so the
    per-sweep rounding differences add up to ~1e-12), same iteration count,
    policy equal up to near-ties."""
    m = pvi.make_preset(preset).set_algorithm("factored")
    res = pvi.run_value_iteration(m)
    key = f"solve|{preset}|f64"
    it, conv = GOLD[key + "|meta"]
    assert abs(res.iterations - int(it)) <= 1 and res.converged == bool(conv)
    np.testing.assert_allclose(res.values, GOLD[key + "|values"], rtol=1e-9, atol=1e-9)
    _near_tie_ok(pvi, preset, res.values, res.policy, GOLD[key + "|policy"], rel=1e-8)


@pytest.mark.parametrize("preset", ["a/m5/exp5", "a/m5/exp6", "a/m4/exp3", "a/m3/exp8"])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_factored_a_full_sweep_close_to_exact(pvi, preset, prec):
    exact = pvi.make_preset(preset)
    fact = pvi.make_preset(preset).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(17).uniform(-40.0, 40.0, n)
    ve, ae = pvi.bellman_backup_batch(exact, V, 0, n, precision=prec)
    vf, af = pvi.bellman_backup_batch(fact, V, 0, n, precision=prec)
    tol = 1e-12 if prec == "f64" else 2e-6
    np.testing.assert_allclose(vf.astype(np.float64), ve.astype(np.float64), rtol=tol, atol=tol * 10)
    if prec == "f64":
        bad = np.nonzero(af != ae)[0]
        assert len(bad) <= max(1, n // 10000)
        for s in bad:
            q = pvi.q_rows(exact, V, int(s), int(s) + 1)[0]
            assert abs(q[af[s]] - q[ae[s]]) <= 1e-9 * max(1.0, abs(q[ae[s]]))
    for s in np.random.default_rng(18).integers(0, n, 8):
        np.testing.assert_allclose(pvi.q_rows(fact, V, int(s), int(s) + 1, precision=prec),
                                   pvi.q_rows(exact, V, int(s), int(s) + 1, precision=prec),
                                   rtol=tol, atol=tol * 10)


def test_factored_b_host_buffer_pipelines_agree(pvi):
    """pvi_vi_backup with host buffers (the e2e leg): the first full-range
    call runs the quarter-piece pipeline, later ones the x_3-pair pipeline
    (V uploaded in 2-D blocks, stage 1 / stage 2 / copy-back per pair).
    Both must equal the device-resident sweep bit for bit."""
    m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(21).uniform(-8.0, 8.0, n)
    v1, a1 = pvi.bellman_backup_batch(m, V, 0, n)
    v2, a2 = pvi.bellman_backup_batch(m, V, 0, n)
    np.testing.assert_array_equal(v1, v2)
    np.testing.assert_array_equal(a1, a2)
    # a sub-range call (no pipeline) agrees on its states
    lo, hi = 5 * 4096 * 256 + 77, 9 * 4096 * 256 + 5
    v3, a3 = pvi.bellman_backup_batch(m, V, lo, hi)
    np.testing.assert_array_equal(v3, v2[lo:hi])
    np.testing.assert_array_equal(a3, a2[lo:hi])


@pytest.mark.parametrize("preset,parts", [("b/m3/exp1", 8), ("b/m3/exp1", 3), ("b/m3/exp1", 5)])
def test_shard_reads_only_its_runs(pvi, preset, parts):
    """pvi_sweep_read_runs is what the sharded driver refreshes between
    sweeps: with every V entry OUTSIDE a shard's runs set to NaN, the
    shard's backup must be unchanged (and finite)."""
    m = pvi.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(8).uniform(-20.0, 20.0, n)
    bounds = [int(b) for b in m.partition(parts)]
    for r in sorted({0, parts // 2, parts - 1}):
        lo, hi = bounds[r], bounds[r + 1]
        runs = m.sweep_read_runs(lo, hi)
        covered = sum(b - a for a, b in runs)
        assert covered < n  # the factored B sweep of a shard reads part of V
        assert all(a < b for a, b in runs) and all(runs[i][1] < runs[i + 1][0] for i in range(len(runs) - 1))
        Vp = np.full(n, np.nan)
        for a, b in runs:
            Vp[a:b] = V[a:b]
        v0, a0 = pvi.bellman_backup_batch(m, V, lo, hi)
        v1, a1 = pvi.bellman_backup_batch(m, Vp, lo, hi)
        assert np.isfinite(v1).all()
        np.testing.assert_array_equal(v1, v0)
        np.testing.assert_array_equal(a1, a0)


def test_read_runs_whole_space_for_gather_sweeps(pvi):
    for preset, algo in [("b/m3/exp4", "exact"), ("c/m5/exp1", "exact"), ("a/m5/exp5", "factored")]:
        m = pvi.make_preset(preset).set_algorithm(algo)
        n = m.state_count()
        assert m.sweep_read_runs(n // 3, n // 2) == [(0, n)]


@pytest.mark.parametrize("max_order,slopes", [(22, [0.0, 0.0]), (22, [0.4, -0.2]), (14, [0.0, 0.0]),
                                              (25, [0.3, 0.1])])
def test_factored_c_other_radix_close_to_exact(pvi, max_order, slopes):
    """Factored C at A_max != 20 (radix r = A_max + 1): the r = 21-templated
    passes (k_c_bin_tile_p<21>, k_c_bin_qf<21>) must step aside for the
    generic ones (k_c_bin_tile_p<0> for r <= 21, k_c_bin_level above it) and
    k_c_bin_qf, which maps 256 threads onto 12 groups of r states, must not
    run for r > 21 (states x_1 >= 14 kept stale values at r = 22)."""
    kw = dict(useful_life=3, max_order=max_order, max_demand=20, life_slopes=slopes)
    exact = pvi.ScenarioC(**kw)
    fact = pvi.ScenarioC(**kw).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(23).uniform(-30.0, 30.0, n)
    ve, ae = pvi.bellman_backup_batch(exact, V, 0, n)
    vf, af = pvi.bellman_backup_batch(fact, V, 0, n)
    np.testing.assert_allclose(vf, ve, rtol=1e-12, atol=1e-10)
    bad = np.nonzero(af != ae)[0]
    for s in bad:
        q = pvi.q_rows(exact, V, int(s), int(s) + 1)[0]
        assert abs(q[af[s]] - q[ae[s]]) <= 1e-9 * max(1.0, abs(q[ae[s]]))
    # and a converged solve
    re = pvi.run_value_iteration(exact)
    rf = pvi.run_value_iteration(fact)
    assert re.iterations == rf.iterations
    np.testing.assert_allclose(rf.values, re.values, rtol=1e-9)


@pytest.mark.parametrize("preset", ["c/m5/exp1", "c/m5/exp2"])
def test_factored_c_weekday_shard_reads_only_its_runs(pvi, preset):
    """A factored-C weekday shard computes only its weekdays' tables: with
    every V entry outside its read runs (own weekdays + the next weekday's
    slice) set to NaN, its backup is unchanged."""
    m = pvi.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(8).uniform(-20.0, 20.0, n)
    full_v, full_a = pvi.bellman_backup_batch(m, V, 0, n)
    b = [int(x) for x in m.partition(3)]
    for r in range(3):
        lo, hi = b[r], b[r + 1]
        Vp = np.full(n, np.nan)
        for x, y in m.sweep_read_runs(lo, hi):
            Vp[x:y] = V[x:y]
        v, a = pvi.bellman_backup_batch(m, Vp, lo, hi)
        np.testing.assert_array_equal(v, full_v[lo:hi])
        np.testing.assert_array_equal(a, full_a[lo:hi])


@pytest.mark.parametrize("preset,algo", [("c/m5/exp1", "factored"), ("b/m3/exp4", "exact"),
                                         ("a/m5/exp5", "factored")])
def test_empty_range_sweep_has_neutral_statistics(pvi, preset, algo):
    """A rank that owns no state (7 weekdays over 8 ranks) still reports
    neutral statistics for the MAX all-reduce: -DBL_MAX everywhere, in
    particular no 'first non-finite state 0' from stale buffers."""
    import torch
    m = pvi.make_preset(preset).set_algorithm(algo)
    n = m.state_count()
    v = torch.zeros(n, dtype=torch.float64, device="cuda")
    vn = torch.empty_like(v)
    st = torch.full((4,), 123.0, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    # poison the rank-local statistics buffer with a real sweep first
    pvi.sweep_device(m, "f64", m.discount(), v.data_ptr(), vn.data_ptr(), None, 0, min(n, 4096),
                     "change_span", (), st.data_ptr(), s)
    pvi.sweep_device(m, "f64", m.discount(), v.data_ptr(), vn.data_ptr(), None, n, n, "change_span", (),
                     st.data_ptr(), s)
    torch.cuda.synchronize()
    got = st.cpu().numpy()
    assert (got[:3] == -1.7976931348623157e308).all(), got


@pytest.mark.parametrize("slopes", [[0.0, 0.0, 0.0], [0.4, -0.2, 0.1]])
def test_factored_c_m4_radix21_close_to_exact(pvi, slopes):
    """useful_life = 4 at A_max = D_max = 20: the r = 21 kernels with other
    line shapes than the presets -- the DMMA G convolution for M = 4, the
    wide DMMA pass for k = 3 with a single x_2-batched line per weekday and
    order (endogenous law, slopes != 0) or the scalar anti-diagonal pass
    (exogenous), then the fused last pass + Q."""
    kw = dict(useful_life=4, max_order=20, max_demand=20, life_slopes=slopes)
    exact = pvi.ScenarioC(**kw)
    fact = pvi.ScenarioC(**kw).set_algorithm("factored")
    n = exact.state_count()
    V = np.random.default_rng(29).uniform(-30.0, 30.0, n)
    ve, ae = pvi.bellman_backup_batch(exact, V, 0, n)
    vf, af = pvi.bellman_backup_batch(fact, V, 0, n)
    np.testing.assert_allclose(vf, ve, rtol=1e-12, atol=1e-10)
    for s in np.nonzero(af != ae)[0]:
        q = pvi.q_rows(exact, V, int(s), int(s) + 1)[0]
        assert abs(q[af[s]] - q[ae[s]]) <= 1e-9 * max(1.0, abs(q[ae[s]]))
    qe = pvi.q_rows(exact, V, n // 3, n // 3 + 200)
    qf = pvi.q_rows(fact, V, n // 3, n // 3 + 200)
    np.testing.assert_allclose(qf, qe, rtol=1e-12, atol=1e-10)
    re = pvi.run_value_iteration(exact)
    rf = pvi.run_value_iteration(fact)
    assert re.iterations == rf.iterations
    np.testing.assert_allclose(rf.values, re.values, rtol=1e-9)
