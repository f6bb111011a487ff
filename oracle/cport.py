"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the C restatement
(oracle/pvi_oracle.c -> oracle/liboracle.so).

The restatement is the checker that travels with the repo: it needs no
/root/reference, so the GPU parity tests and __graft_entry__.smoke() can
compare the CUDA path with it anywhere.  It is itself pinned to the
compiled reference and to tests/golden/ by tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_vp = C.c_void_p
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.orc_preset.restype = _vp
        L.orc_preset.argtypes = [C.c_char_p]
        L.orc_free.argtypes = [_vp]
        L.orc_states.restype = C.c_uint64
        L.orc_states.argtypes = [_vp]
        L.orc_actions.restype = C.c_uint32
        L.orc_actions.argtypes = [_vp]
        L.orc_gamma.restype = C.c_double
        L.orc_gamma.argtypes = [_vp]
        L.orc_backup_range.argtypes = [_vp, C.c_int, _vp, C.c_uint64, C.c_uint64, _vp, _vp]
        L.orc_q_row.argtypes = [_vp, C.c_int, C.c_uint64, _vp, _vp]
        L.orc_initial_values.argtypes = [_vp, _vp]
        L.orc_vi_solve.argtypes = [_vp, C.c_int, C.c_uint64, C.c_uint64, C.c_double, _vp, _vp,
                                   _vp, _vp, _vp]
        L.orc_rollouts.argtypes = [_vp, C.c_int, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                   C.c_uint64, _vp]
        L.orc_reduce.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
        L.orc_philox.argtypes = [_vp, _vp, _vp]
        _lib = L
    return _lib


def available() -> bool:
    return os.path.exists(LIB_PATH)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Model:
    def __init__(self, preset: str):
        self.h = lib().orc_preset(preset.encode())
        if not self.h:
            raise ValueError(f"unknown preset {preset}")
        self.states = lib().orc_states(self.h)
        self.actions = lib().orc_actions(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free(self.h)
            self.h = None


_cache: dict = {}


def model(preset: str) -> Model:
    if preset not in _cache:
        _cache[preset] = Model(preset)
    return _cache[preset]


def backup_range(preset: str, values, lo: int, hi: int, f32: bool = False):
    m = model(preset)
    v = np.ascontiguousarray(values, np.float64)
    ov = np.zeros(hi - lo, np.float64)
    oa = np.zeros(hi - lo, np.uint32)
    lib().orc_backup_range(m.h, int(f32), _p(v), lo, hi, _p(ov), _p(oa))
    return ov, oa


def q_row(preset: str, s: int, values, f32: bool = False):
    m = model(preset)
    v = np.ascontiguousarray(values, np.float64)
    q = np.zeros(m.actions, np.float64)
    lib().orc_q_row(m.h, int(f32), s, _p(v), _p(q))
    return q


def initial_values(preset: str):
    m = model(preset)
    out = np.zeros(m.states, np.float64)
    lib().orc_initial_values(m.h, _p(out))
    return out


class Solve:
    def __init__(self, values, policy, iterations, converged):
        self.values, self.policy, self.iterations, self.converged = values, policy, iterations, converged


def vi_solve(preset: str, f32: bool = False, fixed_iterations: int = 0,
             max_iterations: int = 10000, epsilon: float = 1e-4) -> Solve:
    m = model(preset)
    V = np.zeros(m.states, np.float64)
    P = np.zeros(m.states, np.uint32)
    it, conv, ei = C.c_uint64(), C.c_int(), C.c_uint64()
    rc = lib().orc_vi_solve(m.h, int(f32), fixed_iterations, max_iterations, epsilon, _p(V),
                            _p(P), C.byref(it), C.byref(conv), C.byref(ei))
    if rc:
        raise RuntimeError(f"numeric divergence at iteration {ei.value}")
    return Solve(V, P, it.value, bool(conv.value))


def _rollouts(preset, kind, table, params, n, horizon, warmup, seed):
    m = model(preset)
    out = np.zeros((n, 7), np.float64)
    t = None if table is None else np.ascontiguousarray(table, np.uint32)
    p = np.zeros(14, np.int32)
    if params is not None:
        p[:len(params)] = params
    rc = lib().orc_rollouts(m.h, kind, _p(t), _p(p), n, horizon, warmup, seed, _p(out))
    if rc:
        raise RuntimeError("policy returned an out-of-range order")
    return out


def eval_heuristic(preset: str, params, n_rollouts: int, horizon: int = 365, warmup: int = 100,
                   seed: int = 42):
    return _rollouts(preset, 1, None, params, n_rollouts, horizon, warmup, seed)


def eval_table(preset: str, table, n_rollouts: int, horizon: int = 365, warmup: int = 100,
               seed: int = 42):
    return _rollouts(preset, 0, table, None, n_rollouts, horizon, warmup, seed)


def reduce(xs) -> tuple:
    a = np.ascontiguousarray(xs, np.float64)
    mean, sd = C.c_double(), C.c_double()
    lib().orc_reduce(_p(a), len(a), 1, C.byref(mean), C.byref(sd))
    return mean.value, sd.value


def philox(ctr, key):
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(out))
    return out
