"""C-ABI boundary checks that need no GPU: the library loads and exports
every symbol include/pvi_b200.h declares; host-side models (tables,
cardinalities, fingerprints, index arithmetic, transitions) match the
reference; error taxonomy and checkpoint format.  Compute calls are not
made here except to confirm they fail loudly without a device."""
import ctypes
import hashlib
import os
import re

import numpy as np
import pytest

import paper_2303_10672_b200 as P
from paper_2303_10672_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pvi_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pvi_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes signature table covers all of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def test_version_and_exit_codes():
    assert "sm_100a" in P.version()
    # runner.cpp:482-498 mapping
    assert [P.exit_code(s) for s in (0, 1, 2, 3, 4, 5, 6, 10, 11)] == [0, 1, 2, 3, 4, 5, 1, 2, 1]


# acceptance_main.cpp:90-104 cardinalities
CARDS = [("a/m2/exp1", 121, 11, 101), ("a/m2/exp5", 1331, 11, 101), ("a/m3/exp1", 1331, 11, 101),
         ("a/m3/exp5", 14641, 11, 101), ("a/m4/exp1", 14641, 11, 101),
         ("a/m4/exp5", 161051, 11, 101), ("a/m5/exp1", 161051, 11, 101),
         ("a/m5/exp5", 1771561, 11, 101), ("b/m2/exp1", 14641, 121, 441),
         ("b/m2/exp2", 11025, 105, 377), ("b/m3/exp1", 16777216, 256, 2116),
         ("b/m3/exp2", 10648000, 220, 1792), ("b/m3/exp3", 7529536, 196, 1600),
         ("b/m3/exp4", 1157625, 105, 793), ("b/m2/p1", 14641, 121, 441),
         ("b/m2/p2", 20449, 143, 525), ("b/m2/p3", 28561, 169, 625),
         ("b/m2/p4", 38416, 196, 729), ("c/m3/exp1", 3087, 21, 37191),
         ("c/m3/exp2", 3087, 21, 37191), ("c/m5/exp1", 1361367, 21, 1115730)]


@pytest.mark.parametrize("preset,ns,na,no", CARDS)
def test_cardinalities(preset, ns, na, no):
    m = P.make_preset(preset)
    assert (m.state_count(), m.action_count(), m.outcome_count()) == (ns, na, no)


def test_terms_per_sweep_closed_forms():
    # SURVEY §8d
    assert P.make_preset("a/m2/exp1").terms_per_sweep() == 121 * 11 * 101
    assert P.make_preset("b/m3/exp1").terms_per_sweep() == 2371895689216.0
    assert P.make_preset("c/m5/exp1").terms_per_sweep() == 1361367 * 21 * 53130


def test_tables_bitwise_equal_reference():
    m = P.make_preset("a/m2/exp1")
    np.testing.assert_array_equal(m.table("a.pmf"), GOLD["table|a/m2/exp1|a.pmf"])
    for preset in ["b/m2/exp1", "b/m3/exp1", "b/m3/exp4"]:
        m = P.make_preset(preset)
        for k in ["pu", "pz", "pz_cum"]:
            np.testing.assert_array_equal(m.table(f"b.{k}"), GOLD[f"table|{preset}|b.{k}"])
        caps = GOLD[f"table|{preset}|caps"]
        assert (m.info.max_order_a, m.info.max_order_b) == tuple(caps)
    for preset in ["c/m3/exp1", "c/m3/exp2", "c/m5/exp1", "c/m5/exp2"]:
        m = P.make_preset(preset)
        np.testing.assert_array_equal(m.table("c.pmf"), GOLD[f"table|{preset}|c.pmf"])
        np.testing.assert_array_equal(m.table("c.comp_probs"), GOLD[f"table|{preset}|c.comp_probs"])


def test_gamma_pmf_frozen_values():
    # test_dist.cpp:43-60 (50-digit quadrature, 1e-10)
    p = P.make_preset("a/m2/exp1").table("a.pmf")
    assert p[0] == pytest.approx(0.0017516225562908236521, rel=1e-10)
    assert p[4] == pytest.approx(0.19433671206619395465, rel=1e-10)
    assert sum(p) == 1.0
    assert len(p) == 101


def test_negbinom_frozen_values():
    # test_dist.cpp:105-123 and test_scenario_c.cpp:54-68
    p = P.make_preset("c/m3/exp1").table("c.pmf").reshape(7, 21)
    assert p[0, 0] == pytest.approx(0.033961022655604473532, rel=1e-12)
    assert p[0, 2] == pytest.approx(0.10266097359858980497, rel=1e-12)
    assert p[0, 7] == pytest.approx(0.080522976496274564691, rel=1e-12)
    assert p[6, 0] == pytest.approx(0.12803132451497213352, rel=1e-12)


def test_receipt_probabilities_frozen():
    # test_scenario_c.cpp:25-52
    r = P.make_preset("c/m3/exp1").table("c.receipt_probs").reshape(21, 3)
    assert r[0, 0] == pytest.approx(0.18632372322584757702, rel=1e-13)
    assert r[0, 1] == pytest.approx(0.5064803910556540259, rel=1e-13)
    assert r[0, 2] == pytest.approx(0.30719588571849839707, rel=1e-13)


def test_fingerprint_is_sha256_of_material():
    m = P.make_preset("b/m3/exp1")
    assert m.fingerprint_material() == ("scenario=b;m=3;mu_a=5;mu_b=5;A_a_max=15;A_b_max=15;"
                                        "C_v_a=0.5;C_v_b=0.5;C_r_a=1;C_r_b=1;rho=0.5;gamma=1")
    assert m.fingerprint() == hashlib.sha256(m.fingerprint_material().encode()).digest()
    assert P.sha256(b"abc").hex() == hashlib.sha256(b"abc").hexdigest()


def test_encode_decode_roundtrip_and_bounds():
    m = P.make_preset("b/m2/exp1")
    for s in [0, 1, 777, 14640]:
        assert m.encode(m.decode(s)) == s
    with pytest.raises(P.IndexingError):
        m.encode([11, 0, 0, 0])


def test_worked_transitions_scenario_a():
    # test_scenario_a.cpp:24-40
    fifo = P.ScenarioA(issuing="fifo")
    lifo = P.ScenarioA(issuing="lifo")
    s = fifo.encode([3, 2])
    nf, rf = fifo.transition(s, 4, 1)
    assert fifo.decode(nf) == [4, 3] and rf == -22.0
    nl, rl = lifo.transition(s, 4, 1)
    assert lifo.decode(nl) == [4, 2] and rl == -28.0
    lead2 = P.ScenarioA(issuing="fifo", lead_time=2)
    n2, r2 = lead2.transition(lead2.encode([6, 0, 0]), 2, 0)
    assert lead2.decode(n2) == [2, 6, 0] and r2 == -6.0


def test_worked_transition_scenario_c_capacity_rejection():
    # test_scenario_c.cpp:117-136
    m = P.make_preset("c/m3/exp1")
    s = m.encode([0, 0, 20])
    comp = m.outcome_count() // 21
    # find the composition (0, 0, 3): three expiring units
    found = None
    for w in range(comp):
        try:
            nxt, r = m.transition(s, 3, w)
        except P.ContractViolation:
            continue
        if r == -10.0 - 20.0 - 5.0 * 20.0 and m.decode(nxt) == [1, 0, 0]:
            found = w
            break
    assert found is not None
    with pytest.raises(P.ContractViolation):
        m.transition(s, 2, found)


def test_host_naive_q_row_matches_reference_naive_oracle():
    """naive_q_row (tests/support/oracles.hpp:19-32) over the host transition
    model reproduces the reference's naive oracle for the sampled states."""
    for preset in ["a/m5/exp5", "b/m3/exp4"]:
        m = P.make_preset(preset)
        states = GOLD[f"qrow|{preset}|states"][:1]
        V = np.random.default_rng(7).uniform(-5.0, 5.0, m.state_count())
        want = GOLD[f"qrow|{preset}|naive"][0]
        s = int(states[0])
        q = np.zeros(m.action_count())
        for a in range(m.action_count()):
            for w in range(m.outcome_count()):
                p = m.outcome_probability(s, a, w)
                if p == 0.0:
                    continue
                nxt, r = m.transition(s, a, w)
                q[a] += p * (r + m.discount() * V[nxt])
        np.testing.assert_array_equal(q, want)


def test_capacity_gate_before_any_device_work():
    # c/m8 is refused with the required count (acceptance_main.cpp:368-385)
    m = P.make_preset("c/m8/exp1")
    assert m.state_count() == 12607619787
    with pytest.raises(P.CapacityError) as e:
        P.run_value_iteration(m)
    assert e.value.required_count == 12607619787
    assert P.exit_code(e.value.status) == 3
    with pytest.raises(P.ParameterError):
        P.run_value_iteration(P.make_preset("a/m2/exp1"), P.ViConfig(epsilon=0.0))


def test_unknown_preset_is_config_error():
    with pytest.raises(P.ConfigError):
        P.make_preset("z/m9/exp9")
    with pytest.raises(P.ParameterError):
        P.ScenarioB(substitution_prob=1.5)


@pytest.mark.skipif(P.device_count() > 0, reason="checks the no-device path")
def test_no_cpu_fallback():
    m = P.make_preset("a/m2/exp1")
    with pytest.raises(P.DeviceError):
        P.run_value_iteration(m)
    with pytest.raises(P.DeviceError):
        P.bellman_backup_batch(m, np.zeros(121), 0, 121)
    with pytest.raises(P.DeviceError):
        P.evaluate_policy(m, P.make_heuristic_policy(m, [5]), P.RolloutConfig(n_rollouts=4))


def test_checkpoint_roundtrip_and_refusals(tmp_path):
    # test_vi.cpp:149-175
    path = str(tmp_path / "ck.ckpt")
    values = np.array([1.0, -2.5, 3.25e-300, 7.125e300, 0.1])
    fp = P.sha256(b"model-under-test")
    P.save_checkpoint(path, values, 42, fp)
    ck = P.load_checkpoint(path, fp)
    assert ck.iteration == 42
    np.testing.assert_array_equal(ck.values, values)
    raw = open(path, "rb").read()
    assert raw[:4] == b"PVI1" and len(raw) == 52 + 40
    with pytest.raises(P.FingerprintMismatch):
        P.load_checkpoint(path, P.sha256(b"model-with-other-params"))
    open(path, "wb").write(b"PVI1trunc")
    with pytest.raises(P.FormatError):
        P.load_checkpoint(path)
    open(path, "wb").write(b"NOPE")
    with pytest.raises(P.FormatError):
        P.load_checkpoint(path)
    with pytest.raises(P.IoError):
        P.load_checkpoint(str(tmp_path / "missing.ckpt"))


def test_partition_is_cost_weighted_and_tile_aligned():
    m = P.make_preset("b/m3/exp1")
    b = [int(x) for x in m.partition(8)]
    assert b[0] == 0 and b[-1] == m.state_count()
    assert all(x % 256 == 0 for x in b)
    import sys
    sys.argv = ["x"]
    import bench
    work = bench.work_from_model(m)
    assert work.terms == m.terms_per_sweep()
    assert abs(work.range_terms(0, m.state_count()) - work.terms) <= 1e-9 * work.terms
    costs = [work.range_terms(b[i], b[i + 1]) for i in range(8)]
    assert max(costs) / (sum(costs) / 8) < 1.01  # equal-count sharding gives 1.30


def test_sweep_read_runs_host_logic(pvi):
    """pvi_sweep_read_runs needs no device: factored B x_3-pair shards read
    their own rows' slabs, the lower pairs' constants rows and their own
    states; everything else reads all of V."""
    m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
    n = m.state_count()
    b = [int(x) for x in m.partition(8)]
    assert b == [i * n // 8 for i in range(9)]  # one x_3 pair per shard
    slab = 16 ** 3
    for r in range(8):
        runs = m.sweep_read_runs(b[r], b[r + 1])
        cover = sum(y - x for x, y in runs)
        # own pair rows (32 slabs per top digit) + constants rows of lower
        # pairs (2r per top digit) + own states, minus their overlap
        want = (16 * (32 + 2 * r) + 256 * 2 - 2 * (32 + 2 * r)) * slab
        assert cover == want, (r, cover, want)
    assert pvi.make_preset("b/m3/exp1").sweep_read_runs(0, 5) == [(0, n)]


def test_factored_c_weekday_shards_host_logic(pvi):
    """Factored C: shards are whole weekdays and a weekday shard reads only
    V's next-weekday slices plus its own states (launch_c_factored)."""
    for preset in ["c/m5/exp1", "c/m3/exp2"]:
        m = pvi.make_preset(preset).set_algorithm("factored")
        n = m.state_count()
        w = n // 7
        for parts, sizes in [(2, [4, 3]), (3, [3, 2, 2]), (4, [2, 2, 2, 1]), (7, [1] * 7), (8, [1] * 7 + [0])]:
            b = [int(x) for x in m.partition(parts)]
            assert [(b[i + 1] - b[i]) // w for i in range(parts)] == sizes and b[-1] == n
        for t in range(7):
            nt = (t + 1) % 7
            runs = m.sweep_read_runs(t * w, (t + 1) * w)
            want = sorted([(t * w, (t + 1) * w), (nt * w, (nt + 1) * w)])
            if want[0][1] == want[1][0]:
                want = [(want[0][0], want[1][1])]
            assert runs == want, (preset, t, runs)
        # the exact kernels gather from anywhere
        assert pvi.make_preset(preset).sweep_read_runs(0, w) == [(0, n)]


def test_reference_arm_work_model_matches_product():
    """bench.py's reference arm derives the term counts from oracle/_ref alone
    (it must not load this package): same closed forms as the product's."""
    import sys
    sys.argv = ["x"]
    import bench
    from oracle import refbind
    if not refbind.available():
        pytest.skip("oracle/_ref not built")
    for preset in ["b/m3/exp1", "b/m2/exp1", "c/m5/exp1", "a/m5/exp5", "b/m3/exp4"]:
        a = bench.work_from_reference(preset)
        b = bench.work_from_model(P.make_preset(preset))
        assert (a.states, a.actions) == (b.states, b.actions)
        assert abs(a.terms - b.terms) <= 1e-9 * b.terms, preset
        lo, hi = b.states // 3, b.states // 3 + 4096
        assert a.range_terms(lo, hi) == b.range_terms(lo, hi)
