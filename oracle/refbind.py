"""TEST INFRASTRUCTURE ONLY — ctypes bindings to oracle/_ref/libpvi_ref.so.

That library is the unmodified reference (/root/reference/proj) compiled by
oracle/Makefile plus the C entry points in oracle/ref_capi.cpp.  Only
tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libpvi_ref.so")

_u64p = C.POINTER(C.c_uint64)
_vp = C.c_void_p
_lib = None


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str, value: int = 0):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg
        self.value = value


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        E = [C.c_char_p, C.c_size_t]
        L.ref_model_counts.argtypes = [C.c_char_p, _vp, _vp, _vp, _vp] + E
        L.ref_vi_solve.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                                   C.c_double, C.c_uint64, _vp, _vp, _vp, _vp, _vp] + E
        L.ref_backup_range.argtypes = [C.c_char_p, C.c_int, C.c_int, _vp, C.c_uint64, C.c_uint64,
                                       _vp, _vp, _vp] + E
        L.ref_q_row.argtypes = [C.c_char_p, C.c_int, C.c_uint64, _vp, _vp] + E
        L.ref_naive_q_row.argtypes = [C.c_char_p, C.c_uint64, _vp, _vp] + E
        L.ref_initial_values.argtypes = [C.c_char_p, _vp] + E
        L.ref_eval_heuristic.argtypes = [C.c_char_p, _vp, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_uint64, C.c_int, _vp, _vp] + E
        L.ref_eval_table.argtypes = [C.c_char_p, _vp, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                     C.c_int, _vp, _vp] + E
        L.ref_simopt.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, C.c_int, _vp, _vp,
                                 _vp, _vp, _vp, C.c_int, _vp, _vp, _vp] + E
        L.ref_table_a_pmf.argtypes = [C.c_char_p, _vp] + E
        L.ref_b_issued_pmf.argtypes = [C.c_char_p, C.c_uint64, _vp] + E
        L.ref_b_tables.argtypes = [C.c_char_p, _vp, _vp, _vp, _vp] + E
        L.ref_c_tables.argtypes = [C.c_char_p, _vp, _vp, _vp, _vp] + E
        L.ref_tabular_random.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                         C.c_uint64, _vp, _vp, _vp]
        L.ref_tabular_solve.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double, _vp, _vp,
                                        _vp, _vp, C.c_int, C.c_uint64, C.c_uint64, C.c_double,
                                        C.c_uint64, _vp, _vp, _vp, _vp, _vp] + E
        L.ref_tabular_brute_force.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                              _vp, _vp, _vp, _vp, _vp]
        L.ref_philox_block.argtypes = [_vp, _vp, _vp]
        L.ref_rollout_draws.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, _vp]
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int, err, value: int = 0):
    if rc != 0:
        raise RefError(rc, err.value.decode(errors="replace"), value)


def _err():
    return C.create_string_buffer(1024)


def hardware_threads() -> int:
    return lib().ref_hardware_threads()


@dataclass
class Counts:
    states: int
    actions: int
    outcomes: int
    gamma: float


def counts(preset: str) -> Counts:
    ns, na, no, g = C.c_uint64(), C.c_uint32(), C.c_uint64(), C.c_double()
    e = _err()
    _check(lib().ref_model_counts(preset.encode(), C.byref(ns), C.byref(na), C.byref(no),
                                  C.byref(g), e, len(e)), e)
    return Counts(ns.value, na.value, no.value, g.value)


@dataclass
class Solve:
    values: np.ndarray
    policy: np.ndarray
    iterations: int
    converged: bool
    wall_seconds: float


def vi_solve(preset: str, f32: bool = False, threads: int | None = None,
             fixed_iterations: int = 0, max_iterations: int = 10000, epsilon: float = 1e-4,
             max_batch: int = 0) -> Solve:
    n = counts(preset).states
    V = np.zeros(n, np.float64)
    P = np.zeros(n, np.uint32)
    it, conv, wall = C.c_uint64(), C.c_int(), C.c_double()
    e = _err()
    _check(lib().ref_vi_solve(preset.encode(), int(f32), threads or hardware_threads(),
                              fixed_iterations, max_iterations, epsilon, max_batch, _p(V), _p(P),
                              C.byref(it), C.byref(conv), C.byref(wall), e, len(e)), e)
    return Solve(V, P, it.value, bool(conv.value), wall.value)


def backup_range(preset: str, values: np.ndarray, lo: int, hi: int, f32: bool = False,
                 threads: int | None = None):
    values = np.ascontiguousarray(values, np.float64)
    ov = np.zeros(hi - lo, np.float64)
    oa = np.zeros(hi - lo, np.uint32)
    secs = C.c_double()
    e = _err()
    _check(lib().ref_backup_range(preset.encode(), int(f32), threads or hardware_threads(),
                                  _p(values), lo, hi, _p(ov), _p(oa), C.byref(secs), e, len(e)), e)
    return ov, oa, secs.value


def q_row(preset: str, state: int, values: np.ndarray, f32: bool = False) -> np.ndarray:
    values = np.ascontiguousarray(values, np.float64)
    q = np.zeros(counts(preset).actions, np.float64)
    e = _err()
    _check(lib().ref_q_row(preset.encode(), int(f32), state, _p(values), _p(q), e, len(e)), e)
    return q


def naive_q_row(preset: str, state: int, values: np.ndarray) -> np.ndarray:
    values = np.ascontiguousarray(values, np.float64)
    q = np.zeros(counts(preset).actions, np.float64)
    e = _err()
    _check(lib().ref_naive_q_row(preset.encode(), state, _p(values), _p(q), e, len(e)), e)
    return q


def initial_values(preset: str) -> np.ndarray:
    out = np.zeros(counts(preset).states, np.float64)
    e = _err()
    _check(lib().ref_initial_values(preset.encode(), _p(out), e, len(e)), e)
    return out


def eval_heuristic(preset: str, params, n_rollouts: int, horizon: int = 365, warmup: int = 100,
                   seed: int = 42, threads: int | None = None, per_rollout: bool = True):
    p = np.ascontiguousarray(params, np.int32)
    pr = np.zeros((n_rollouts, 7), np.float64) if per_rollout else None
    ev = np.zeros(14, np.float64)
    e = _err()
    _check(lib().ref_eval_heuristic(preset.encode(), _p(p), len(p), n_rollouts, horizon, warmup,
                                    seed, threads or hardware_threads(), _p(pr), _p(ev), e,
                                    len(e)), e)
    return pr, ev


def eval_table(preset: str, actions: np.ndarray, n_rollouts: int, horizon: int = 365,
               warmup: int = 100, seed: int = 42, threads: int | None = None,
               per_rollout: bool = True):
    a = np.ascontiguousarray(actions, np.uint32)
    pr = np.zeros((n_rollouts, 7), np.float64) if per_rollout else None
    ev = np.zeros(14, np.float64)
    e = _err()
    _check(lib().ref_eval_table(preset.encode(), _p(a), n_rollouts, horizon, warmup, seed,
                                threads or hardware_threads(), _p(pr), _p(ev), e, len(e)), e)
    return pr, ev


def simopt(preset: str, rollouts: int = 4096, eval_seed: int = 42, ga_seed: int = 1,
           threads: int | None = None, max_log: int = 20000):
    dim = 14
    best = np.zeros(dim, np.int32)
    bm, bsd, wall = C.c_double(), C.c_double(), C.c_double()
    gens, nlog = C.c_int(), C.c_int()
    lv = np.zeros(max_log * dim, np.int32)
    ls = np.zeros(max_log * 3, np.float64)
    e = _err()
    _check(lib().ref_simopt(preset.encode(), rollouts, eval_seed, ga_seed,
                            threads or hardware_threads(), _p(best), C.byref(bm), C.byref(bsd),
                            C.byref(gens), C.byref(nlog), max_log, _p(lv), _p(ls),
                            C.byref(wall), e, len(e)), e)
    return dict(best=best, mean=bm.value, sd=bsd.value, generations=gens.value,
                n_logged=nlog.value, log_values=lv, log_scores=ls.reshape(-1, 3)[: nlog.value],
                wall=wall.value)


def table_a_pmf(preset: str, d_max: int = 100) -> np.ndarray:
    out = np.zeros(d_max + 1, np.float64)
    e = _err()
    _check(lib().ref_table_a_pmf(preset.encode(), _p(out), e, len(e)), e)
    return out


def b_issued_pmf(preset: str, state: int) -> np.ndarray:
    out = np.zeros(counts(preset).outcomes, np.float64)
    e = _err()
    _check(lib().ref_b_issued_pmf(preset.encode(), state, _p(out), e, len(e)), e)
    return out


def b_tables(preset: str):
    caps = np.zeros(4, np.int32)
    e = _err()
    _check(lib().ref_b_tables(preset.encode(), _p(caps), None, None, None, e, len(e)), e)
    d_max, y_max = int(caps[2]), int(caps[3])
    shape = (y_max + 1, d_max + 1)
    pu, pz, pzc = (np.zeros(shape, np.float64) for _ in range(3))
    _check(lib().ref_b_tables(preset.encode(), _p(caps), _p(pu), _p(pz), _p(pzc), e, len(e)), e)
    return dict(max_order_a=int(caps[0]), max_order_b=int(caps[1]), d_max=d_max, y_max=y_max,
                pu=pu, pz=pz, pz_cum=pzc)


def c_tables(preset: str, max_order: int = 20, max_demand: int = 20):
    wk = np.zeros((7, max_demand + 1), np.float64)
    off = np.zeros(max_order + 2, np.uint32)
    e = _err()
    _check(lib().ref_c_tables(preset.encode(), _p(wk), _p(off), None, None, e, len(e)), e)
    total = int(off[-1])
    ids = np.zeros(total, np.uint32)
    probs = np.zeros(total, np.float64)
    _check(lib().ref_c_tables(preset.encode(), _p(wk), _p(off), _p(ids), _p(probs), e, len(e)), e)
    return dict(weekday_pmf=wk, offsets=off, ids=ids, probs=probs)


def tabular_random(ns: int, na: int, no: int, gamma: float, seed: int):
    size = ns * na * no
    nxt = np.zeros(size, np.uint64)
    rew = np.zeros(size, np.float64)
    prob = np.zeros(size, np.float64)
    lib().ref_tabular_random(ns, na, no, gamma, seed, _p(nxt), _p(rew), _p(prob))
    return nxt, rew, prob


def tabular_solve(ns, na, no, gamma, nxt, rew, prob, initial=None, f32=False,
                  fixed_iterations=0, max_iterations=10000, epsilon=1e-4,
                  max_states=200_000_000):
    V = np.zeros(ns, np.float64)
    P = np.zeros(ns, np.uint32)
    it, conv, ev = C.c_uint64(), C.c_int(), C.c_uint64()
    e = _err()
    init = None if initial is None else np.ascontiguousarray(initial, np.float64)
    rc = lib().ref_tabular_solve(ns, na, no, gamma, _p(nxt), _p(rew), _p(prob), _p(init),
                                 int(f32), fixed_iterations, max_iterations, epsilon, max_states,
                                 _p(V), _p(P), C.byref(it), C.byref(conv), C.byref(ev), e, len(e))
    _check(rc, e, ev.value)
    return Solve(V, P, it.value, bool(conv.value), 0.0)


def tabular_brute_force(ns, na, no, gamma, nxt, rew, prob):
    V = np.zeros(ns, np.float64)
    P = np.zeros(ns, np.uint32)
    lib().ref_tabular_brute_force(ns, na, no, gamma, _p(nxt), _p(rew), _p(prob), _p(V), _p(P))
    return V, P


def philox_block(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().ref_philox_block(_p(c), _p(k), _p(out))
    return out


def rollout_draws(seed: int, rollout: int, day: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    lib().ref_rollout_draws(seed, rollout, day, n, _p(out))
    return out
