"""Graph-resident sweep loop and the persisting L2 window (pvi_vi_config
loop / l2_persist).

The loop control of run_value_iteration (vi.hpp:220-265: non-finite check,
convergence test, iteration limit) runs on the device after every sweep and
drives a CUDA-graph WHILE node, so a solve is one graph launch.  It must
change nothing: iteration counts, values and policies are bit-identical to
the host-driven loop (and so to the reference, tests/test_gpu_vi.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(pvi, preset, **kw):
    m = pvi.make_preset(preset)
    algo = kw.pop("algorithm", None)
    if algo:
        m.set_algorithm(algo)
    return pvi.run_value_iteration(m, pvi.ViConfig(**kw))


def _same(a, b):
    assert (a.iterations, a.converged) == (b.iterations, b.converged)
    np.testing.assert_array_equal(a.values, b.values)
    np.testing.assert_array_equal(a.policy, b.policy)
    assert (a.span_lo, a.span_hi) == (b.span_lo, b.span_hi)


@pytest.mark.parametrize("preset,kw", [
    ("a/m2/exp1", {}),
    ("a/m2/exp1", {"precision": "f32"}),
    ("a/m3/exp1", {}),
    ("a/m2/exp1", {"algorithm": "factored"}),
    ("b/m2/exp1", {}),
    ("b/m2/exp1", {"algorithm": "factored"}),
    ("b/m2/p1", {"fixed_iterations": 100}),
    ("a/m2/exp1", {"max_iterations": 37}),
    ("c/m3/exp1", {}),
    ("c/m3/exp1", {"algorithm": "factored"}),
    ("c/m3/exp2", {"algorithm": "factored"}),
    ("c/m3/exp1", {"precision": "f32"}),
    ("c/m3/exp1", {"max_iterations": 12}),
    ("c/m3/exp1", {"fixed_iterations": 20}),
])
def test_graph_loop_equals_host_loop(pvi, preset, kw):
    host = _solve(pvi, preset, loop="host", **dict(kw))
    graph = _solve(pvi, preset, loop="graph", **dict(kw))
    _same(host, graph)
    assert host.graph_sweeps == 0
    # the first sweep runs eagerly (periodic span: the 7 that fill the 8-slot ring)
    eager = 7 if preset.startswith("c/") else 1
    assert graph.graph_sweeps == graph.iterations - eager


def test_graph_loop_periodic_matches_reference(pvi):
    # the 8-slot ring (a chain of IF nodes per phase) reproduces the reference's c/m3 solves bit for bit
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
    for preset in ("c/m3/exp1", "c/m3/exp2"):
        key = f"solve|{preset}|f64"
        r = _solve(pvi, preset, loop="graph")
        assert r.graph_sweeps == r.iterations - 7
        it, conv = gold[key + "|meta"]
        assert r.iterations == it and r.converged == bool(conv)
        np.testing.assert_array_equal(r.values, gold[key + "|values"])
        np.testing.assert_array_equal(r.policy, gold[key + "|policy"])


def test_graph_loop_limits(pvi):
    r = _solve(pvi, "a/m2/exp1", loop="graph", max_iterations=37)
    assert r.iterations == 37 and not r.converged
    r = _solve(pvi, "b/m2/p1", loop="graph", fixed_iterations=100)
    assert r.iterations == 100 and r.converged


def test_graph_loop_divergence(pvi):
    # test_vi.cpp:225-240 through the graph: the second sweep overflows
    m = pvi.TabularMdp(2, 1, 1, 1.0, [0, 1], [1e308, 1e308], [1.0, 1.0])
    with pytest.raises(pvi.NumericDivergence) as e:
        pvi.run_value_iteration(m, pvi.ViConfig(fixed_iterations=10, loop="graph"))
    assert e.value.iteration == 2 and "state 0" in str(e.value)


def test_graph_loop_refuses_unsupported(pvi, tmp_path):
    with pytest.raises(pvi.ParameterError):
        _solve(pvi, "a/m2/exp1", loop="graph", checkpoint_every=100,
               checkpoint_path=str(tmp_path / "c.ckpt"))
    # auto: the host loop with checkpoints, and for the periodic span (its
    # 8-branch graph is built only on request); the graph otherwise
    r = _solve(pvi, "a/m2/exp1", checkpoint_every=100, checkpoint_path=str(tmp_path / "d.ckpt"))
    assert r.graph_sweeps == 0 and r.converged
    r = _solve(pvi, "c/m3/exp1")
    assert r.graph_sweeps == 0 and r.converged
    r = _solve(pvi, "a/m2/exp1")
    assert r.graph_sweeps == r.iterations - 1 and r.converged


def test_l2_window_auto(pvi):
    # auto: a window over the value ring for the exact kernels only
    assert _solve(pvi, "a/m2/exp1", algorithm="exact").l2_window_bytes > 0
    assert _solve(pvi, "a/m2/exp1", algorithm="factored").l2_window_bytes == 0


@pytest.mark.parametrize("preset", ["a/m3/exp1", "b/m2/exp1", "c/m3/exp1"])
def test_l2_window_changes_nothing(pvi, preset):
    on = _solve(pvi, preset, l2_persist=True)
    off = _solve(pvi, preset, l2_persist=False)
    _same(on, off)
    assert off.l2_window_bytes == 0
    assert on.l2_window_bytes > 0 and 0.0 < on.l2_hit_ratio <= 1.0
