"""Python mirror of the reference's solver / simulator API over the C ABI.

Names, argument meaning and error behaviour follow the reference C++
library (proj/include/pvi/*.hpp) so that the parity tests read like the
reference's own tests:

  ScenarioA/B/C(params)            scenario_{a,b,c}.hpp constructors
  TabularMdp(...)                  tests/support/tabular_mdp.hpp
  make_preset(name)                presets.cpp:82-130
  run_value_iteration(model, cfg)  vi.hpp:295-302
  bellman_backup_batch(...)        vi.hpp:82-92
  check_convergence(...)           vi.hpp:107-158
  evaluate_policy(model, policy, cfg) / evaluate_policies(...)   sim.hpp:145-170
  make_vi_policy / make_heuristic_policy                         policies.hpp:18-82

Exceptions mirror errors.hpp:11-57.  Every compute call runs on the GPU
through libpvi_b200.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

# ---------------------------------------------------------------------------
# errors (errors.hpp:11-57)


class Error(RuntimeError):
    status = 1


class ParameterError(Error):
    status = 2


class ConfigError(Error):
    status = 10


class IndexingError(Error):
    status = 9


class ContractViolation(Error):
    status = 6


class IoError(Error):
    status = 5


class FormatError(Error):
    status = 7


class FingerprintMismatch(Error):
    status = 8


class DeviceError(Error):
    status = 11


class CapacityError(Error):
    status = 3

    def __init__(self, msg: str, required_count: int):
        super().__init__(msg)
        self.required_count = required_count


class NumericDivergence(Error):
    status = 4

    def __init__(self, msg: str, iteration: int):
        super().__init__(msg)
        self.iteration = iteration


_BY_STATUS = {c.status: c for c in (Error, ParameterError, ConfigError, IndexingError,
                                     ContractViolation, IoError, FormatError,
                                     FingerprintMismatch, DeviceError)}

VALUE_SPAN, CHANGE_SPAN, PERIODIC_SPAN = 0, 1, 2
_TEST_NAMES = {"value_span": 0, "change_span": 1, "periodic_span": 2}
_ALGOS = {"exact": 0, "factored": 1}


def _err_buf():
    return C.create_string_buffer(2048)


def _raise(rc: int, err, value: int = 0):
    if rc == 0:
        return
    msg = err.value.decode(errors="replace") if err is not None else f"status {rc}"
    if rc == CapacityError.status:
        raise CapacityError(msg, value)
    if rc == NumericDivergence.status:
        raise NumericDivergence(msg, value)
    raise _BY_STATUS.get(rc, Error)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def exit_code(status: int) -> int:
    return L.load().pvi_exit_code(status)


def device_count() -> int:
    return L.load().pvi_device_count()


def version() -> str:
    return L.load().pvi_version().decode()


# ---------------------------------------------------------------------------
# parameters


def scenario_a_params(**kw) -> L.ScenarioAParams:
    p = L.ScenarioAParams()
    L.load().pvi_scenario_a_defaults(C.byref(p))
    for k, v in kw.items():
        if k == "issuing" and isinstance(v, str):
            v = 0 if v == "fifo" else 1
        setattr(p, k, v)
    return p


def scenario_b_params(**kw) -> L.ScenarioBParams:
    p = L.ScenarioBParams()
    L.load().pvi_scenario_b_defaults(C.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def scenario_c_params(**kw) -> L.ScenarioCParams:
    p = L.ScenarioCParams()
    L.load().pvi_scenario_c_defaults(C.byref(p))
    for k, v in kw.items():
        if k in ("demand_successes", "demand_means", "life_intercepts", "life_slopes"):
            arr = getattr(p, k)
            for i in range(len(arr)):
                arr[i] = 0.0
            for i, x in enumerate(v):
                arr[i] = x
        else:
            setattr(p, k, v)
    return p


# ---------------------------------------------------------------------------
# models


class Model:
    """An immutable MDP (MdpModel + Simulator concepts, model.hpp:30-46, sim.hpp:25-35)."""

    def __init__(self, handle: C.c_void_p, name: str = "custom", fixed_iterations: int = 0,
                 checkpoint_every: int = 0):
        self._h = handle
        self.name = name
        self.preset_fixed_iterations = fixed_iterations
        self.preset_checkpoint_every = checkpoint_every
        info = L.ModelInfo()
        _raise(L.load().pvi_model_get_info(self._h, C.byref(info)), None)
        self.info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                L.load().pvi_model_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    # model contract
    def state_count(self) -> int:
        return int(self.info.state_count)

    def action_count(self) -> int:
        return int(self.info.action_count)

    def outcome_count(self) -> int:
        return int(self.info.outcome_count)

    def discount(self) -> float:
        return float(self.info.discount)

    def default_convergence_test(self) -> int:
        return int(self.info.default_convergence_test)

    def periodicity(self) -> int:
        return int(self.info.periodicity)

    def state_arity(self) -> int:
        return int(self.info.state_arity)

    def products(self) -> int:
        return int(self.info.products)

    def terms_per_sweep(self) -> float:
        return float(self.info.terms_per_sweep)

    def scenario(self) -> str:
        return "abct"[self.info.scenario]

    def fingerprint_material(self) -> str:
        buf = C.create_string_buffer(4096)
        _raise(L.load().pvi_model_fingerprint_material(self._h, buf, len(buf)), None)
        return buf.value.decode()

    def fingerprint(self) -> bytes:
        out = (C.c_uint8 * 32)()
        _raise(L.load().pvi_model_fingerprint(self._h, out), None)
        return bytes(out)

    def table(self, name: str) -> np.ndarray:
        n = C.c_size_t()
        lib = L.load()
        _raise(lib.pvi_model_table(self._h, name.encode(), None, C.byref(n)), None)
        out = np.zeros(n.value, np.float64)
        _raise(lib.pvi_model_table(self._h, name.encode(), _p(out), C.byref(n)), None)
        return out

    def decode(self, index: int) -> list:
        out = np.zeros(self.state_arity(), np.int32)
        _raise(L.load().pvi_model_decode(self._h, index, _p(out)), None)
        return [int(x) for x in out]

    def encode(self, tup: Sequence[int]) -> int:
        t = np.ascontiguousarray(tup, np.int32)
        idx = C.c_uint64()
        err = _err_buf()
        _raise(L.load().pvi_model_encode(self._h, _p(t), C.byref(idx), err, len(err)), err)
        return idx.value

    def transition(self, s: int, a: int, w: int):
        nxt, rew = C.c_uint64(), C.c_double()
        err = _err_buf()
        _raise(L.load().pvi_model_transition(self._h, s, a, w, C.byref(nxt), C.byref(rew), err,
                                             len(err)), err)
        return nxt.value, rew.value

    def outcome_probability(self, s: int, a: int, w: int) -> float:
        p = C.c_double()
        _raise(L.load().pvi_model_outcome_probability(self._h, s, a, w, C.byref(p)), None)
        return p.value

    def initial_values(self) -> np.ndarray:
        out = np.zeros(self.state_count(), np.float64)
        err = _err_buf()
        _raise(L.load().pvi_model_initial_values(self._h, _p(out), err, len(err)), err)
        return out

    def set_algorithm(self, algorithm: str) -> "Model":
        """'exact' (reference order, bit-identical) or 'factored' (Scenario B:
        separable issued-pair contraction, agrees to rounding)."""
        _raise(L.load().pvi_model_set_algorithm(self._h, _ALGOS[algorithm]), None)
        self.algorithm = algorithm
        return self

    def partition(self, parts: int) -> np.ndarray:
        b = np.zeros(parts + 1, np.uint64)
        _raise(L.load().pvi_partition(self._h, parts, _p(b)), None)
        return b

    def policy_csv_body(self, actions: np.ndarray) -> bytes:
        """The rows of runner.cpp's policy_to_csv (one per state, no header),
        formatted on the device (pvi_policy_csv_format)."""
        a = np.ascontiguousarray(actions, np.uint32)
        if a.shape != (self.state_count(),):
            raise ParameterError("policy must have one action per state")
        ln = C.c_uint64()
        err = _err_buf()
        _raise(L.load().pvi_policy_csv_format(self._h, _p(a), None, 0, C.byref(ln), err, len(err)), err)
        buf = np.empty(ln.value, np.uint8)
        _raise(L.load().pvi_policy_csv_format(self._h, _p(a), _p(buf), ln.value, C.byref(ln), err, len(err)), err)
        return buf.tobytes()

    def policy_from_csv_text(self, text: bytes) -> np.ndarray:
        """runner.cpp's policy_from_csv after the metadata check, parsed on
        the device (pvi_policy_csv_parse)."""
        out = np.zeros(self.state_count(), np.uint32)
        buf = np.frombuffer(text, np.uint8)
        err = _err_buf()
        _raise(L.load().pvi_policy_csv_parse(self._h, _p(buf) if len(buf) else None, len(buf), _p(out), err,
                                             len(err)), err)
        return out

    def unit_count(self) -> int:
        """Units of the factored B x_3-pair sweep (pvi_unit_count)."""
        c = C.c_uint64()
        _raise(L.load().pvi_unit_count(self._h, C.byref(c)), None)
        return int(c.value)

    def unit_partition(self, parts: int) -> np.ndarray:
        b = np.zeros(parts + 1, np.uint64)
        _raise(L.load().pvi_unit_partition(self._h, parts, _p(b)), None)
        return b

    def unit_runs(self, u_lo: int, u_hi: int, read: bool = False) -> list:
        """State runs of a unit shard: its own states, or (read=True) what its
        sweep reads (pvi_unit_runs)."""
        cnt = C.c_size_t()
        w = 1 if read else 0
        _raise(L.load().pvi_unit_runs(self._h, u_lo, u_hi, w, None, 0, C.byref(cnt)), None)
        buf = np.zeros(2 * cnt.value, np.uint64)
        _raise(L.load().pvi_unit_runs(self._h, u_lo, u_hi, w, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                      cnt.value, C.byref(cnt)), None)
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt.value)]

    def sweep_read_runs(self, lo: int, hi: int) -> list:
        """State runs [(a, b), ...] of V that a sweep of shard [lo, hi) reads
        (pvi_sweep_read_runs): what a multi-GPU driver must refresh."""
        cnt = C.c_size_t()
        _raise(L.load().pvi_sweep_read_runs(self._h, lo, hi, None, 0, C.byref(cnt)), None)
        buf = np.zeros(2 * cnt.value, np.uint64)
        _raise(L.load().pvi_sweep_read_runs(self._h, lo, hi, buf.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            cnt.value, C.byref(cnt)), None)
        return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt.value)]


def _create(fn, params) -> C.c_void_p:
    h = C.c_void_p()
    err = _err_buf()
    _raise(fn(C.byref(params), C.byref(h), err, len(err)), err)
    return h


def ScenarioA(params: Optional[L.ScenarioAParams] = None, **kw) -> Model:
    p = params if params is not None else scenario_a_params(**kw)
    return Model(_create(L.load().pvi_model_create_a, p))


def ScenarioB(params: Optional[L.ScenarioBParams] = None, **kw) -> Model:
    p = params if params is not None else scenario_b_params(**kw)
    return Model(_create(L.load().pvi_model_create_b, p))


def ScenarioC(params: Optional[L.ScenarioCParams] = None, **kw) -> Model:
    p = params if params is not None else scenario_c_params(**kw)
    return Model(_create(L.load().pvi_model_create_c, p))


def TabularMdp(n_states: int, n_actions: int, n_outcomes: int, gamma: float, next_state,
               reward, prob, initial=None) -> Model:
    nxt = np.ascontiguousarray(next_state, np.uint64)
    rew = np.ascontiguousarray(reward, np.float64)
    pr = np.ascontiguousarray(prob, np.float64)
    ini = None if initial is None else np.ascontiguousarray(initial, np.float64)
    h = C.c_void_p()
    err = _err_buf()
    _raise(L.load().pvi_model_create_tabular(n_states, n_actions, n_outcomes, gamma, _p(nxt),
                                             _p(rew), _p(pr), _p(ini), C.byref(h), err,
                                             len(err)), err)
    return Model(h, "tabular")


def make_preset(name: str) -> Model:
    h = C.c_void_p()
    fixed, every = C.c_uint64(), C.c_uint64()
    err = _err_buf()
    _raise(L.load().pvi_model_create_preset(name.encode(), C.byref(h), C.byref(fixed),
                                            C.byref(every), err, len(err)), err)
    return Model(h, name, fixed.value, every.value)


def preset_names() -> list:
    names = [f"a/m{m}/exp{e}" for m in range(2, 6) for e in range(1, 9)]
    names += ["b/m2/exp1", "b/m2/exp2", "b/m3/exp1", "b/m3/exp2", "b/m3/exp3", "b/m3/exp4",
              "b/m2/p1", "b/m2/p2", "b/m2/p3", "b/m2/p4"]
    names += [f"c/m{m}/exp{e}" for m in (3, 5, 8) for e in (1, 2)]
    return names


# ---------------------------------------------------------------------------
# value iteration (vi.hpp)


@dataclass
class ViConfig:
    epsilon: float = 1e-4
    gamma: Optional[float] = None
    max_iterations: int = 10_000
    fixed_iterations: int = 0
    checkpoint_every: int = 0
    checkpoint_path: str = ""
    precision: str = "f64"
    convergence_test: Optional[str] = None
    max_states: int = 200_000_000
    device: int = -1
    algorithm: Optional[str] = None  # None: the model's (Model.set_algorithm)
    loop: str = "auto"               # "auto" | "host" | "graph" (pvi_vi_config::loop)
    l2_persist: Optional[bool] = None  # None: auto (on for the exact kernels)

    def to_c(self) -> L.ViConfigC:
        c = L.ViConfigC()
        L.load().pvi_vi_config_defaults(C.byref(c))
        c.epsilon = self.epsilon
        if self.gamma is not None:
            c.gamma = self.gamma
            c.has_gamma = 1
        c.max_iterations = self.max_iterations
        c.fixed_iterations = self.fixed_iterations
        c.checkpoint_every = self.checkpoint_every
        self._path = self.checkpoint_path.encode() if self.checkpoint_path else None
        c.checkpoint_path = self._path
        c.precision = 1 if self.precision == "f32" else 0
        c.convergence_test = -1 if self.convergence_test is None else _TEST_NAMES[self.convergence_test]
        c.max_states = self.max_states
        c.device = self.device
        c.algorithm = -1 if self.algorithm is None else _ALGOS[self.algorithm]
        c.loop = {"auto": -1, "host": 0, "graph": 1}[self.loop]
        c.l2_persist = -1 if self.l2_persist is None else int(bool(self.l2_persist))
        return c


@dataclass
class Checkpoint:
    values: np.ndarray
    iteration: int
    fingerprint: bytes


@dataclass
class ViResult:
    values: np.ndarray          # ValueFunction::values (f64)
    policy: np.ndarray          # Policy::actions (u32)
    iterations: int
    converged: bool
    wall_seconds: float
    sweep_seconds: float = 0.0
    sweeps: int = 0
    span_lo: float = 0.0
    span_hi: float = 0.0
    terms_per_sweep: float = 0.0
    fingerprint: bytes = b""
    graph_sweeps: int = 0        # sweeps inside the graph-resident loop
    l2_window_bytes: int = 0     # persisting L2 access-policy window
    l2_hit_ratio: float = 0.0


def run_value_iteration(model: Model, config: Optional[ViConfig] = None,
                        resume: Optional[Checkpoint] = None) -> ViResult:
    config = config or ViConfig()
    n = model.state_count()
    fits = n <= config.max_states  # else the C side raises CapacityError first
    # value-initialised like the reference's std::vector results (pages
    # touched here, so the device-to-host copy does not page-fault)
    values = np.empty(n, np.float64) if fits else None
    policy = np.empty(n, np.uint32) if fits else None
    if fits:
        values.fill(0.0)
        policy.fill(0)
    st = L.ViStats()
    ev = C.c_uint64()
    err = _err_buf()
    cc = config.to_c()
    rv = rf = None
    rit = 0
    if resume is not None:
        if len(resume.values) != n:
            raise FormatError(f"resume checkpoint has {len(resume.values)} states, model has {n}")
        rv = np.ascontiguousarray(resume.values, np.float64)
        rf = (C.c_uint8 * 32).from_buffer_copy(resume.fingerprint)
        rit = resume.iteration
    rc = L.load().pvi_vi_solve(model.handle, C.byref(cc), _p(rv), rit,
                               None if rf is None else C.byref(rf), _p(values), _p(policy),
                               C.byref(st), C.byref(ev), err, len(err))
    _raise(rc, err, ev.value)
    return ViResult(values, policy, int(st.iterations), bool(st.converged), st.wall_seconds,
                    st.sweep_seconds, int(st.sweeps), st.span_lo, st.span_hi,
                    st.terms_per_sweep, model.fingerprint(), int(st.graph_sweeps),
                    int(st.l2_window_bytes), float(st.l2_hit_ratio))


def _dtype(precision: str):
    return np.float32 if precision == "f32" else np.float64


def sweep_device(model: Model, precision: str, gamma: float, vprev_ptr: int, vnext_ptr: int,
                 actions_ptr: Optional[int], lo: int, hi: int, test: Optional[str] = None,
                 hist_ptrs: Sequence[int] = (), stats_ptr: Optional[int] = None,
                 stream_ptr: Optional[int] = None):
    """One device-resident sweep of states [lo, hi) (pvi_vi_sweep_device).

    Pointers are raw device addresses (e.g. torch.Tensor.data_ptr()); the
    launch is asynchronous on `stream_ptr` (a cudaStream_t, e.g.
    torch.cuda.current_stream().cuda_stream)."""
    t = -1 if test is None else _TEST_NAMES[test]
    hist = (C.c_void_p * max(1, len(hist_ptrs)))(*[int(p) for p in hist_ptrs])
    err = _err_buf()
    _raise(L.load().pvi_vi_sweep_device(model.handle, int(precision == "f32"), gamma,
                                        C.c_void_p(vprev_ptr), C.c_void_p(vnext_ptr),
                                        None if actions_ptr is None else C.c_void_p(actions_ptr),
                                        lo, hi, t, hist, len(hist_ptrs),
                                        int(stats_ptr is not None),
                                        None if stats_ptr is None else C.c_void_p(stats_ptr),
                                        None if stream_ptr is None else C.c_void_p(stream_ptr),
                                        err, len(err)), err)


def sweep_device_peers(model: Model, precision: str, gamma: float, vprev_ptr: int, vnext_ptr: int,
                       lo: int, hi: int, peers: Sequence[tuple], test: Optional[str] = None,
                       stats_ptr: Optional[int] = None, stream_ptr: Optional[int] = None):
    """sweep_device with the exchange fused in (pvi_vi_sweep_device_peers):
    `peers` = [(peer_vnext_ptr, peer_lo, peer_hi), ...], the peers' next-value
    buffers mapped into this process (ipc_open) and their shards."""
    t = -1 if test is None else _TEST_NAMES[test]
    n = len(peers)
    ptrs = (C.c_void_p * max(1, n))(*[int(p[0]) for p in peers])
    plo = (C.c_uint64 * max(1, n))(*[int(p[1]) for p in peers])
    phi = (C.c_uint64 * max(1, n))(*[int(p[2]) for p in peers])
    err = _err_buf()
    _raise(L.load().pvi_vi_sweep_device_peers(model.handle, int(precision == "f32"), gamma,
                                              C.c_void_p(vprev_ptr), C.c_void_p(vnext_ptr), lo, hi, t,
                                              int(stats_ptr is not None),
                                              None if stats_ptr is None else C.c_void_p(stats_ptr),
                                              None if stream_ptr is None else C.c_void_p(stream_ptr),
                                              n, ptrs, plo, phi, err, len(err)), err)


def sweep_device_units(model: Model, gamma: float, vprev_ptr: int, vnext_ptr: int, u_lo: int, u_hi: int,
                       peers: Sequence[tuple] = (), test: Optional[str] = None,
                       stats_ptr: Optional[int] = None, stream_ptr: Optional[int] = None,
                       actions_ptr: Optional[int] = None):
    """The sweep of unit shard [u_lo, u_hi) (pvi_vi_sweep_device_units, f64),
    optionally storing into peers' replicas: peers = [(ptr, peer_u_lo, peer_u_hi)]."""
    t = -1 if test is None else _TEST_NAMES[test]
    n = len(peers)
    ptrs = (C.c_void_p * max(1, n))(*[int(p[0]) for p in peers])
    plo = (C.c_uint64 * max(1, n))(*[int(p[1]) for p in peers])
    phi = (C.c_uint64 * max(1, n))(*[int(p[2]) for p in peers])
    err = _err_buf()
    _raise(L.load().pvi_vi_sweep_device_units(model.handle, 0, gamma, C.c_void_p(vprev_ptr),
                                              C.c_void_p(vnext_ptr),
                                              None if actions_ptr is None else C.c_void_p(actions_ptr),
                                              u_lo, u_hi, t, int(stats_ptr is not None),
                                              None if stats_ptr is None else C.c_void_p(stats_ptr),
                                              None if stream_ptr is None else C.c_void_p(stream_ptr),
                                              n, ptrs, plo, phi, err, len(err)), err)


class DeviceBuffer:
    """A cudaMalloc'd device buffer (pvi_device_alloc) that other processes
    can map (ipc_handle / ipc_open); usable from torch through
    __cuda_array_interface__ (torch.as_tensor(buf, device="cuda"))."""

    def __init__(self, count: int, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.count = int(count)
        p = C.c_void_p()
        err = _err_buf()
        _raise(L.load().pvi_device_alloc(self.count * self.dtype.itemsize, C.byref(p), err, len(err)), err)
        self.ptr = int(p.value)

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.count,), "typestr": self.dtype.str, "data": (self.ptr, False),
                "version": 3, "strides": None}

    def ipc_handle(self) -> bytes:
        h = (C.c_uint8 * 64)()
        err = _err_buf()
        _raise(L.load().pvi_ipc_get_handle(C.c_void_p(self.ptr), h, err, len(err)), err)
        return bytes(h)

    def free(self):
        if self.ptr:
            L.load().pvi_device_free(C.c_void_p(self.ptr))
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def ipc_open(handle: bytes) -> int:
    """Map a peer process's DeviceBuffer (by its 64-byte handle) into this
    process; returns the device pointer (ipc_close to unmap)."""
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    err = _err_buf()
    _raise(L.load().pvi_ipc_open(h, C.byref(p), err, len(err)), err)
    return int(p.value)


def ipc_close(ptr: int):
    _raise(L.load().pvi_ipc_close(C.c_void_p(ptr)), None)


def profile_enable(on: bool = True):
    _raise(L.load().pvi_profile_enable(int(on)), None)


def profile_sim_read():
    """(philox_blocks, rollout_days, kernel_ms) of the evaluations since the last read
    (pvi_profile_sim_read; counted while profile_enable(True))."""
    b, d, ms = C.c_uint64(), C.c_uint64(), C.c_double()
    _raise(L.load().pvi_profile_sim_read(C.byref(b), C.byref(d), C.byref(ms)), None)
    return b.value, d.value, ms.value


def profile_read():
    """(K1 milliseconds, K1 launches, all VI-path kernel launches) since enable/read."""
    ms, k, a = C.c_double(), C.c_uint64(), C.c_uint64()
    _raise(L.load().pvi_profile_read(C.byref(ms), C.byref(k), C.byref(a)), None)
    return ms.value, k.value, a.value


def bellman_backup_batch(model: Model, values, lo: int, hi: int, gamma: Optional[float] = None,
                         precision: str = "f64", out_values: Optional[np.ndarray] = None,
                         out_actions: Optional[np.ndarray] = None):
    """(values[hi-lo], actions[hi-lo]) of one synchronous backup (vi.hpp:82-92).
    out_values / out_actions may be caller-owned (e.g. pinned) host arrays."""
    dt = _dtype(precision)
    v = np.ascontiguousarray(values, dt)
    ov = np.zeros(hi - lo, dt) if out_values is None else out_values
    oa = np.zeros(hi - lo, np.uint32) if out_actions is None else out_actions
    assert ov.dtype == dt and oa.dtype == np.uint32 and len(ov) == len(oa) == hi - lo
    err = _err_buf()
    g = model.discount() if gamma is None else gamma
    _raise(L.load().pvi_vi_backup(model.handle, int(dt == np.float32), g, _p(v), lo, hi,
                                  _p(ov), _p(oa), err, len(err)), err)
    return ov, oa


def q_rows(model: Model, values, lo: int, hi: int, gamma: Optional[float] = None,
           precision: str = "f64") -> np.ndarray:
    """Q(s, a) for s in [lo, hi) (q_row, model.hpp:25-29)."""
    dt = _dtype(precision)
    v = np.ascontiguousarray(values, dt)
    q = np.zeros((hi - lo, model.action_count()), dt)
    err = _err_buf()
    g = model.discount() if gamma is None else gamma
    _raise(L.load().pvi_q_rows(model.handle, int(dt == np.float32), g, _p(v), lo, hi, _p(q),
                               err, len(err)), err)
    return q


def check_convergence(model: Model, test: str, history: Sequence[np.ndarray], gamma: float,
                      epsilon: float, iteration: int, precision: str = "f64") -> bool:
    dt = _dtype(precision)
    hs = [np.ascontiguousarray(h, dt) for h in history]
    arr = (C.c_void_p * max(1, len(hs)))(*[h.ctypes.data for h in hs])
    conv = C.c_int()
    err = _err_buf()
    _raise(L.load().pvi_check_convergence(model.handle, int(dt == np.float32), _TEST_NAMES[test],
                                          arr, len(hs), gamma, epsilon, iteration,
                                          C.byref(conv), err, len(err)), err)
    return bool(conv.value)


# ---------------------------------------------------------------------------
# checkpoints (checkpoint.hpp)


def sha256(data: bytes) -> bytes:
    out = (C.c_uint8 * 32)()
    buf = C.create_string_buffer(data, len(data))
    _raise(L.load().pvi_sha256(buf, len(data), out), None)
    return bytes(out)


def save_checkpoint(path: str, values, iteration: int, fingerprint: bytes):
    v = np.ascontiguousarray(values, np.float64)
    fp = (C.c_uint8 * 32).from_buffer_copy(fingerprint)
    err = _err_buf()
    _raise(L.load().pvi_checkpoint_save(path.encode(), _p(v), len(v), iteration, fp, err,
                                        len(err)), err)


def load_checkpoint(path: str, expected: Optional[bytes] = None) -> Checkpoint:
    lib = L.load()
    cnt, it = C.c_uint64(), C.c_uint64()
    fp = (C.c_uint8 * 32)()
    exp = None if expected is None else (C.c_uint8 * 32).from_buffer_copy(expected)
    err = _err_buf()
    _raise(lib.pvi_checkpoint_load(path.encode(), exp, None, 0, C.byref(cnt), C.byref(it), fp,
                                   err, len(err)), err)
    vals = np.zeros(cnt.value, np.float64)
    _raise(lib.pvi_checkpoint_load(path.encode(), exp, _p(vals), cnt.value, C.byref(cnt),
                                   C.byref(it), fp, err, len(err)), err)
    return Checkpoint(vals, it.value, bytes(fp))


# ---------------------------------------------------------------------------
# simulation (sim.hpp, policies.hpp)


@dataclass
class RolloutConfig:
    horizon_days: int = 365
    warmup_days: int = 100
    n_rollouts: int = 10_000
    base_seed: int = 0
    device: int = -1

    def to_c(self) -> L.RolloutConfigC:
        c = L.RolloutConfigC()
        c.horizon_days = self.horizon_days
        c.warmup_days = self.warmup_days
        c.n_rollouts = self.n_rollouts
        c.base_seed = self.base_seed
        c.device = self.device
        return c


@dataclass
class Policy:
    """Device policy descriptor (replaces the std::function PolicyFn, sim.hpp:37)."""
    kind: int                     # 0 VI table, 1 heuristic
    table: Optional[np.ndarray] = None
    params: Sequence[int] = field(default_factory=list)


def make_vi_policy(model: Model, actions) -> Policy:
    return Policy(0, np.ascontiguousarray(actions, np.uint32))


def make_heuristic_policy(model: Model, params: Sequence[int]) -> Policy:
    return Policy(1, None, list(params))


def heuristic_space(model: Model):
    """(name, lo, hi) per parameter (policies.hpp:44-59)."""
    sc = model.scenario()
    if sc == "a":
        return [("S", 0, model.info.max_order_a)]
    if sc == "b":
        return [("S_a", 0, 2 * model.info.max_order_a), ("S_b", 0, 2 * model.info.max_order_b)]
    return ([(f"s.{t}", 0, model.info.max_order_a) for t in range(7)] +
            [(f"S.{t}", 0, model.info.max_order_a) for t in range(7)])


@dataclass
class KpiStat:
    mean: float = 0.0
    sd: float = 0.0


@dataclass
class Evaluation:
    ret: KpiStat
    service_pct: list
    wastage_pct: list
    holding_mean: list
    products: int
    n_rollouts: int


def _policies_c(policies: Sequence[Policy]):
    arr = (L.PolicyC * len(policies))()
    keep = []
    for i, p in enumerate(policies):
        arr[i].kind = p.kind
        if p.kind == 0:
            t = np.ascontiguousarray(p.table, np.uint32)
            keep.append(t)
            arr[i].table = t.ctypes.data_as(C.POINTER(C.c_uint32))
        for k, v in enumerate(p.params):
            arr[i].params[k] = int(v)
        arr[i].n_params = len(p.params)
    return arr, keep


def evaluate_policies(model: Model, policies: Sequence[Policy], config: RolloutConfig,
                      per_rollout: bool = False):
    """Batched evaluate_policy on common random numbers.

    Returns (evaluations, summaries) where summaries is None or an array of
    shape (n_policies, n_rollouts, 7): ret, service a/b, wastage a/b, holding a/b.
    """
    arr, keep = _policies_c(policies)
    n = len(policies)
    ev = (L.EvaluationC * max(1, n))()
    summ = np.zeros((n, config.n_rollouts, 7), np.float64) if per_rollout else None
    cc = config.to_c()
    err = _err_buf()
    _raise(L.load().pvi_sim_evaluate(model.handle, arr, n, C.byref(cc), _p(summ), ev, err,
                                     len(err)), err)
    out = []
    for i in range(n):
        e = ev[i]
        out.append(Evaluation(KpiStat(e.ret_mean, e.ret_sd),
                              [KpiStat(e.service_mean[k], e.service_sd[k]) for k in range(2)],
                              [KpiStat(e.wastage_mean[k], e.wastage_sd[k]) for k in range(2)],
                              [KpiStat(e.holding_mean[k], e.holding_sd[k]) for k in range(2)],
                              e.products, e.n_rollouts))
    del keep
    return out, summ


def _evaluation(e) -> "Evaluation":
    return Evaluation(KpiStat(e.ret_mean, e.ret_sd),
                      [KpiStat(e.service_mean[k], e.service_sd[k]) for k in range(2)],
                      [KpiStat(e.wastage_mean[k], e.wastage_sd[k]) for k in range(2)],
                      [KpiStat(e.holding_mean[k], e.holding_sd[k]) for k in range(2)],
                      e.products, e.n_rollouts)


def sim_reduce(summaries: np.ndarray, products: int) -> list:
    """detail::reduce (sim.hpp:128-141) of per-rollout summaries shaped
    (n_policies, n_rollouts, 7), in rollout-index order, on the host
    (pvi_sim_reduce): bit-identical to pvi_sim_evaluate's own reduction."""
    a = np.ascontiguousarray(summaries, np.float64)
    n_pol, n = a.shape[0], a.shape[1]
    ev = (L.EvaluationC * max(1, n_pol))()
    err = _err_buf()
    _raise(L.load().pvi_sim_reduce(_p(a), n_pol, n, products, ev, err, len(err)), err)
    return [_evaluation(ev[i]) for i in range(n_pol)]


def evaluate_policy(model: Model, policy: Policy, config: RolloutConfig) -> Evaluation:
    return evaluate_policies(model, [policy], config)[0][0]


@dataclass
class SimoptResult:
    best: list
    best_mean: float
    best_sd: float
    generations: int
    log: list            # (generation, values, mean, sd) per evaluated candidate, in order
    device_seconds: float
    wall_seconds: float


def simopt(model: Model, sampler: str = "auto", population: int = 50, max_generations: int = 100,
           patience: int = 5, crossover_rate: float = 0.9, mutation_rate: float = 0.0,
           seed: int = 1, rollouts_per_candidate: int = 4000, horizon_days: int = 365,
           warmup_days: int = 100, base_seed: int = 42, device: int = -1,
           log_capacity: int = 20000, score_batch=None) -> SimoptResult:
    """cmd_simopt's search (runner.cpp:352-403): grid (1-D) or GA, batched on the GPU.

    score_batch: optional callable (candidates: int array n x dim) -> (means, sds)
    that replaces the single-device evaluator as the batch point (the sharded
    multi-GPU driver passes one; sharded_sim.py)."""
    import time
    c = L.SimoptConfigC()
    lib = L.load()
    lib.pvi_simopt_config_defaults(C.byref(c))
    c.sampler = {"auto": 0, "grid": 1, "ga": 2, "exhaustive": 3}[sampler]
    c.population, c.max_generations, c.patience = population, max_generations, patience
    c.crossover_rate, c.mutation_rate, c.seed = crossover_rate, mutation_rate, seed
    c.rollouts_per_candidate, c.horizon_days, c.warmup_days = (rollouts_per_candidate,
                                                              horizon_days, warmup_days)
    c.base_seed, c.device = base_seed, device
    cb = None
    failure = []
    if score_batch is not None:
        def _cb(user, cands, n, dim, means, sds):
            try:
                arr = np.ctypeslib.as_array(cands, shape=(n * dim,)).reshape(n, dim).copy()
                mu, sd = score_batch(arr)
                for i in range(n):
                    means[i] = float(mu[i])
                    sds[i] = float(sd[i])
                return 0
            except BaseException as e:  # noqa: BLE001 -- reported after the C call returns
                failure.append(e)
                return 1
        cb = L.SCORE_BATCH_FN(_cb)
        c.score_batch = C.cast(cb, C.c_void_p)
    best = (C.c_int * 14)()
    bm, bsd, dev_s = C.c_double(), C.c_double(), C.c_double()
    gens, nlog, dim = C.c_int(), C.c_int(), C.c_int()
    logs = (L.ScoredCandidateC * log_capacity)()
    err = _err_buf()
    t0 = time.perf_counter()
    rc = lib.pvi_simopt(model.handle, C.byref(c), best, C.byref(bm), C.byref(bsd),
                        C.byref(gens), logs, log_capacity, C.byref(nlog), C.byref(dim),
                        C.byref(dev_s), err, len(err))
    if failure:
        raise failure[0]
    _raise(rc, err)
    del cb
    wall = time.perf_counter() - t0
    d = dim.value
    entries = [(logs[i].generation, list(logs[i].values[:d]), logs[i].mean, logs[i].sd)
               for i in range(min(nlog.value, log_capacity))]
    return SimoptResult(list(best[:d]), bm.value, bsd.value, gens.value, entries, dev_s.value,
                        wall)


def philox_block(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    _raise(L.load().pvi_philox_block(_p(c), _p(k), _p(out)), None)
    return out


def rollout_draws(seed: int, rollout: int, day: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    _raise(L.load().pvi_rollout_draws(seed, rollout, day, n, _p(out)), None)
    return out
