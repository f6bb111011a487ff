"""GPU parity of the value-iteration path against the compiled reference.

The device kernels reproduce the reference's per-term arithmetic and
summation order with no FMA contraction, so in f64 AND f32 the value
vectors, iteration counts and policies must be bit-identical to
run_value_iteration (vi.hpp:295) on the same preset.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve_both(pvi, ref, preset, f32=False, **kw):
    m = pvi.make_preset(preset)
    cfg = pvi.ViConfig(precision="f32" if f32 else "f64", **kw)
    got = pvi.run_value_iteration(m, cfg)
    want = ref.vi_solve(preset, f32=f32, fixed_iterations=kw.get("fixed_iterations", 0),
                        max_iterations=kw.get("max_iterations", 10000))
    return got, want


@pytest.mark.parametrize("preset", ["a/m2/exp1", "a/m2/exp2", "a/m2/exp6", "a/m3/exp5",
                                    "b/m2/exp1", "b/m2/exp2", "c/m3/exp1", "c/m3/exp2"])
def test_solve_bitwise_f64(pvi, ref, preset):
    got, want = _solve_both(pvi, ref, preset)
    assert got.iterations == want.iterations
    assert got.converged == want.converged
    np.testing.assert_array_equal(got.values, want.values)
    np.testing.assert_array_equal(got.policy, want.policy)


@pytest.mark.parametrize("preset", ["a/m2/exp1", "c/m3/exp1"])
def test_solve_bitwise_f32(pvi, ref, preset):
    got, want = _solve_both(pvi, ref, preset, f32=True)
    assert got.iterations == want.iterations
    np.testing.assert_array_equal(got.values, want.values)
    np.testing.assert_array_equal(got.policy, want.policy)


def test_fixed_iterations_b_p1(pvi, ref):
    got, want = _solve_both(pvi, ref, "b/m2/p1", fixed_iterations=100)
    assert got.iterations == want.iterations == 100
    np.testing.assert_array_equal(got.values, want.values)
    np.testing.assert_array_equal(got.policy, want.policy)


@pytest.mark.parametrize("preset,states", [("b/m3/exp1", [0, 1, 4095, 65536 * 7 + 1234, 16777215]),
                                           ("c/m5/exp1", [0, 1, 700000, 1361366]),
                                           ("b/m3/exp4", [0, 5000, 1157624])])
def test_q_rows_match_reference(pvi, ref, preset, states):
    m = pvi.make_preset(preset)
    rng = np.random.default_rng(7)
    V = rng.uniform(-5, 5, m.state_count())
    for s in states:
        q = pvi.q_rows(m, V, s, s + 1)[0]
        np.testing.assert_array_equal(q, ref.q_row(preset, s, V))


def test_initial_values_b(pvi, ref):
    m = pvi.make_preset("b/m2/exp1")
    np.testing.assert_array_equal(m.initial_values(), ref.initial_values("b/m2/exp1"))
