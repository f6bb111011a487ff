"""Multi-GPU value iteration: one process per GPU over torch.distributed.

The state space is split into contiguous, cost-weighted shards
(pvi_partition; Scenario B's per-state work is (I_a+1)(I_b+1), so equal
counts would leave the 8-GPU load at 1.30x the mean).  Every
rank holds a full replica of V_prev, backs up its own slice, and the slices
are exchanged with one NCCL all-gather per sweep; the convergence
statistic of each slice (max, -min, first non-finite state) is combined with
one 4-double MAX all-reduce.  Max and min are exact, so the convergence
decision, the iteration count and the value vector are identical to the
single-GPU run (and to the reference).

Read-set exchange.  A sweep of shard [lo, hi) does not always read all of
V: the factored Scenario B sweep of an x_3-pair shard reads ~1/8 of the
value slabs plus its own states (pvi_sweep_read_runs).  Then the per-sweep
refresh is not an all-gather of every slice but ONE uneven all-to-all
(NCCL all_to_all_single over NVLink): rank q sends rank r exactly
runs(r) ∩ [lo_q, hi_q), gathered by one index_select and scattered by one
index_copy_ on each side (index tensors built once).  For b/m3/exp1 at 8
ranks that is ~16 MiB received per rank per sweep instead of 112 MiB.
The full replica is re-assembled (one all-gather) only where a caller needs
all of V: checkpoints and the returned value vector.

Fused exchange (exchange="peer").  The ranks' value buffers are CUDA-IPC
shared (pvi_device_alloc / pvi_ipc_open), and the factored B sweep writes
each finished V' entry straight into the replicas of the peers whose next
sweep reads it, over NVLink peer memory, from the stage-2 finalize
(pvi_vi_sweep_device_peers) -- the exchange overlaps the sweep instead of
following it.  The MAX all-reduce of the statistics is the only collective
left; it also orders every rank's stores before the next sweep.

The per-slice sweep is injectable so the host logic (partition, exchange,
reduction, history window, convergence) runs under `gloo` on CPU in tests;
the default sweep is the device kernel through pvi_vi_sweep_device.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import pvi as P

NEG_INF = -1.7976931348623157e308

SweepFn = Callable[..., None]


def evaluate_test(test: int, hi: float, lo: float, epsilon: float, iteration: int) -> bool:
    """check_convergence's decision from the reduced statistic (vi.hpp:107-158)."""
    if test == P.VALUE_SPAN:
        return max(0.0, hi) < epsilon
    if test == P.CHANGE_SPAN:
        return hi - lo < epsilon
    if iteration < 7:
        return False
    return hi - lo <= 2.0 * epsilon * min(abs(hi), abs(lo))


def device_sweep(model: P.Model, precision: str, gamma: float):
    def sweep(vprev: torch.Tensor, vnext: torch.Tensor, actions: Optional[torch.Tensor],
              lo: int, hi: int, test: Optional[int], hist: List[torch.Tensor],
              stats: Optional[torch.Tensor]):
        names = {0: "value_span", 1: "change_span", 2: "periodic_span"}
        P.sweep_device(model, precision, gamma, vprev.data_ptr(), vnext.data_ptr(),
                       None if actions is None else actions.data_ptr(), lo, hi,
                       None if test is None else names[test], [h.data_ptr() for h in hist],
                       None if stats is None else stats.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    return sweep


@dataclass
class ShardedResult:
    values: np.ndarray
    policy: np.ndarray
    iterations: int
    converged: bool
    wall_seconds: float
    sweep_seconds: float
    bounds: list


class ShardedValueIteration:
    """run_value_iteration (vi.hpp:162-291) over `world` ranks."""

    def __init__(self, model: P.Model, config: Optional[P.ViConfig] = None,
                 device: Optional[torch.device] = None, sweep: Optional[SweepFn] = None,
                 group=None, exchange: str = "auto", shards: str = "auto"):
        """exchange: "auto"/"runs" -- refresh the read set with one NCCL
        all-to-all (all-gather when the sweep reads all of V); "peer" -- the
        sweep itself stores V' into the peers' IPC-mapped replicas (factored
        B x_3-pair sweep on CUDA devices; falls back to "runs" otherwise)."""
        self.model = model
        self.exchange_mode = exchange
        self.cfg = config or P.ViConfig()
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device or (torch.device("cuda", torch.cuda.current_device())
                                 if torch.cuda.is_available() else torch.device("cpu"))
        self.n = model.state_count()
        self.bounds = [int(b) for b in model.partition(self.world)]
        self.lo, self.hi = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.maxlen = max(self.bounds[r + 1] - self.bounds[r] for r in range(self.world))
        # Unit shards (factored B x_3-pair sweep): rank r owns the (pair, x_b
        # column range) blocks of units [ub[r], ub[r+1]) -- balanced finer
        # than whole pairs.  shards: "auto" (units where the sweep supports
        # them and there is more than one rank), "units", "range".
        self.units = None
        test0 = (model.default_convergence_test() if (config is None or config.convergence_test is None)
                 else P._TEST_NAMES[config.convergence_test])
        if shards == "units" and test0 == P.PERIODIC_SPAN:
            raise P.ParameterError("unit shards: the periodic-span statistic needs range shards")
        # the unit sweep has no periodic-span statistic: range shards then
        if shards != "range" and self.world > 1 and test0 != P.PERIODIC_SPAN:
            try:
                nu = model.unit_count()
            except P.Error:
                nu = 0
            if nu and (shards == "units" or sweep is None):
                self.units = [int(b) for b in model.unit_partition(self.world)]
        if self.units is not None:
            ub = self.units
            self.u_lo, self.u_hi = ub[self.rank], ub[self.rank + 1]
            self.own_runs = [model.unit_runs(ub[r], ub[r + 1]) for r in range(self.world)]
            self.read_runs = [model.unit_runs(ub[r], ub[r + 1], read=True) for r in range(self.world)]
        else:
            self.own_runs = [[(self.bounds[r], self.bounds[r + 1])] for r in range(self.world)]
            self.read_runs = None
        self._own_idx = None
        self.dtype = torch.float32 if self.cfg.precision == "f32" else torch.float64
        self.gamma = self.cfg.gamma if self.cfg.gamma is not None else model.discount()
        self.test = (model.default_convergence_test() if self.cfg.convergence_test is None
                     else P._TEST_NAMES[self.cfg.convergence_test])
        self.injected = sweep is not None
        self.sweep = sweep or device_sweep(model, self.cfg.precision, self.gamma)
        self.hist_cap = 8 if self.test == P.PERIODIC_SPAN else 2
        self._send = torch.empty(self.maxlen, dtype=self.dtype, device=self.device)
        self._recv = torch.empty(self.maxlen * self.world, dtype=self.dtype, device=self.device)
        self._setup_read_sets()
        self.peer = None
        self.peer_error = None
        # fused peer stores: factored B sends each entry to the peers that read
        # it; every other sweep (value / change span) broadcasts its slice
        if (exchange == "peer" and self.world > 1 and sweep is None and self.device.type == "cuda"
                and self.test != P.PERIODIC_SPAN):
            self._setup_peers()

    # -- fused peer exchange ---------------------------------------------------
    def _setup_peers(self):
        """Two IPC-shared value buffers per rank; map every peer's pair.
        Every rank must take the same exchange path, so the ranks agree (one
        all-gather of their flags) and all fall back to the read-set all-to-all if any
        of them could not map its peers (e.g. no peer access)."""
        bufs, handles, why = [], [None] * self.world, ""
        try:
            bufs = [P.DeviceBuffer(self.n, np.float32 if self.dtype == torch.float32 else np.float64)
                    for _ in range(2)]
            mine = [b.ipc_handle() for b in bufs]
        except P.Error as e:
            mine, why = None, str(e)
        dist.all_gather_object(handles, mine, group=self.group)
        mapped = [[None] * self.world for _ in range(2)]
        ok = all(h is not None for h in handles)
        if ok:
            try:
                for q in range(self.world):
                    if q != self.rank:
                        for k in range(2):
                            mapped[k][q] = P.ipc_open(handles[q][k])
            except P.Error as e:
                ok, why = False, str(e)
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=self.group)
        if not all(oks):
            for k in range(2):
                for ptr in mapped[k]:
                    if ptr:
                        P.ipc_close(ptr)
            self.peer_error = why or "a peer rank could not map the IPC buffers"
            self.exchange_mode = "runs"
            return
        self.peer = {"bufs": bufs, "tensors": [torch.as_tensor(b, device=self.device) for b in bufs],
                     "mapped": mapped}

    def buffers(self):
        """The two value buffers the fused exchange writes into (peer mode),
        else None: callers that step() with these get the fused path."""
        return None if self.peer is None else tuple(self.peer["tensors"])

    def _peer_slot(self, v: torch.Tensor):
        if self.peer is None:
            return None
        for k, t in enumerate(self.peer["tensors"]):
            if t.data_ptr() == v.data_ptr():
                return k
        return None

    def close(self):
        """Unmap the peers' buffers (collective in peer mode: every rank's
        stores into them are done before any rank unmaps or frees)."""
        if self.peer is not None:
            dist.barrier(group=self.group)
            for k in range(2):
                for q, ptr in enumerate(self.peer["mapped"][k]):
                    if ptr:
                        P.ipc_close(ptr)
            self.peer = None

    # -- the rank's sweep --------------------------------------------------------
    def _sweep(self, vprev, vnext, actions, test, hist, stats, peers=None):
        """This rank's sweep: its state range, or its unit shard."""
        if self.units is None:
            self.sweep(vprev, vnext, actions, self.lo, self.hi, test, list(hist), stats)
            return
        if self.injected:
            self.sweep(vprev, vnext, actions, self.u_lo, self.u_hi, test, list(hist), stats)
            return
        names = {0: "value_span", 1: "change_span"}
        P.sweep_device_units(self.model, self.gamma, vprev.data_ptr(), vnext.data_ptr(), self.u_lo, self.u_hi,
                             peers or (), None if test is None else names[test],
                             None if stats is None else stats.data_ptr(),
                             torch.cuda.current_stream().cuda_stream,
                             None if actions is None else actions.data_ptr())

    # -- read sets -----------------------------------------------------------
    @staticmethod
    def _intersect(ra, rb):
        """Indices in both run lists (sorted, disjoint runs)."""
        out, i, j = [], 0, 0
        while i < len(ra) and j < len(rb):
            a, b = max(ra[i][0], rb[j][0]), min(ra[i][1], rb[j][1])
            if a < b:
                out.append(np.arange(a, b, dtype=np.int64))
            if ra[i][1] < rb[j][1]:
                i += 1
            else:
                j += 1
        return np.concatenate(out) if out else np.zeros(0, np.int64)

    def _setup_read_sets(self):
        """Index plan of the read-set all-to-all (or None: every rank reads
        all of V, so the refresh is the all-gather)."""
        self.plan = None
        if self.world == 1:
            return
        runs = self.read_runs or [self.model.sweep_read_runs(self.bounds[r], self.bounds[r + 1])
                                  for r in range(self.world)]
        if self.units is None and all(rr == [(0, self.n)] for rr in runs):
            return
        me = self.rank
        own = self.own_runs
        send = [self._intersect(runs[q], own[me]) if q != me else np.zeros(0, np.int64)
                for q in range(self.world)]
        recv = [self._intersect(runs[me], own[q]) if q != me else np.zeros(0, np.int64)
                for q in range(self.world)]
        dev = self.device
        self.plan = {
            "send_idx": torch.from_numpy(np.concatenate(send)).to(dev),
            "recv_idx": torch.from_numpy(np.concatenate(recv)).to(dev),
            "send_splits": [len(x) for x in send],
            "recv_splits": [len(x) for x in recv],
            "runs": runs,
        }
        self.plan["recv_buf"] = torch.empty(len(self.plan["recv_idx"]), dtype=self.dtype, device=dev)

    def read_set_bytes(self) -> int:
        """Bytes this rank receives per sweep refresh."""
        if self.world == 1:
            return 0
        item = torch.empty(0, dtype=self.dtype).element_size()
        if self.plan is None:
            return (self.n - (self.hi - self.lo)) * item
        return sum(self.plan["recv_splits"]) * item

    def own_states(self) -> int:
        return sum(b - a for a, b in self.own_runs[self.rank])

    # -- collectives ---------------------------------------------------------
    def exchange(self, v: torch.Tensor, send=None, recv=None):
        """All-gather every rank's slice of `v` into every replica."""
        if self.world == 1:
            return
        if self.units is not None:
            self._exchange_units(v)
            return
        send = self._send if send is None else send
        recv = self._recv if recv is None else recv
        ln = self.hi - self.lo
        send[:ln].copy_(v[self.lo:self.hi])
        dist.all_gather_into_tensor(recv, send, group=self.group)
        for r in range(self.world):
            a, b = self.bounds[r], self.bounds[r + 1]
            if r != self.rank and b > a:
                v[a:b].copy_(recv[r * self.maxlen:r * self.maxlen + (b - a)])

    def _exchange_units(self, v: torch.Tensor):
        """Full-replica all-gather for unit shards (own states are index sets)."""
        if self._own_idx is None:
            idx = [torch.from_numpy(np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in rr]))
                   .to(self.device) for rr in self.own_runs]
            self._own_idx = idx
        idx = self._own_idx
        maxc = max(len(x) for x in idx)
        send = torch.zeros(maxc, dtype=v.dtype, device=v.device)
        send[:len(idx[self.rank])] = v.index_select(0, idx[self.rank])
        recv = torch.empty(maxc * self.world, dtype=v.dtype, device=v.device)
        dist.all_gather_into_tensor(recv, send, group=self.group)
        for q in range(self.world):
            if q != self.rank:
                v.index_copy_(0, idx[q], recv[q * maxc:q * maxc + len(idx[q])])

    def refresh(self, v: torch.Tensor):
        """Make every entry the next sweep of this rank reads current: the
        read-set all-to-all where the sweep reads part of V, else the
        all-gather of the slices."""
        if self.world == 1:
            return
        if self.plan is None:
            self.exchange(v)
            return
        pl = self.plan
        sendbuf = v.index_select(0, pl["send_idx"])
        dist.all_to_all_single(pl["recv_buf"], sendbuf, pl["recv_splits"], pl["send_splits"],
                               group=self.group)
        v.index_copy_(0, pl["recv_idx"], pl["recv_buf"])

    def reduce_stats(self, stats: torch.Tensor):
        if self.world > 1:
            dist.all_reduce(stats, op=dist.ReduceOp.MAX, group=self.group)

    # -- one sweep (bench step) ---------------------------------------------
    def step(self, vprev: torch.Tensor, vnext: torch.Tensor, stats: Optional[torch.Tensor] = None,
             test: Optional[int] = None, hist: List[torch.Tensor] = ()):
        """One sweep + exchange.  `hist` holds the 7 previous vectors
        (oldest..newest, newest = vprev) when test is the periodic span."""
        k = self._peer_slot(vnext)
        if k is not None and test != P.PERIODIC_SPAN:
            self._peer_sweep(vprev, vnext, k, test, stats)
            return
        self._sweep(vprev, vnext, None, test, hist, stats)
        if stats is not None:
            self.reduce_stats(stats)
        self.refresh(vnext)

    def _peer_sweep(self, vprev, vnext, k, test, stats):
        names = {0: "value_span", 1: "change_span"}
        if self.units is not None:
            ub = self.units
            peers = [(self.peer["mapped"][k][q], ub[q], ub[q + 1]) for q in range(self.world) if q != self.rank]
            self._sweep(vprev, vnext, None, test, (), stats, peers)
        else:
            peers = [(self.peer["mapped"][k][q], self.bounds[q], self.bounds[q + 1])
                     for q in range(self.world) if q != self.rank]
            P.sweep_device_peers(self.model, self.cfg.precision, self.gamma, vprev.data_ptr(),
                                 vnext.data_ptr(), self.lo, self.hi, peers,
                                 None if test is None else names[test],
                                 None if stats is None else stats.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream)
        if stats is not None:
            self.reduce_stats(stats)  # also orders every rank's peer stores
        else:
            dist.barrier(group=self.group)

    # -- full solve ----------------------------------------------------------
    def solve(self, resume: Optional[P.Checkpoint] = None) -> ShardedResult:
        t0 = time.perf_counter()
        cfg, n = self.cfg, self.n
        if n > cfg.max_states:
            raise P.CapacityError(f"value iteration requires {n} states, exceeding the "
                                  f"configured capacity of {cfg.max_states}", n)
        if not cfg.epsilon > 0:
            raise P.ParameterError("value iteration: epsilon must be > 0")
        if self.peer is not None and self.hist_cap == 2:
            ring = list(self.peer["tensors"])
        else:
            ring = [torch.empty(n, dtype=self.dtype, device=self.device) for _ in range(self.hist_cap)]
        if resume is not None:
            if resume.fingerprint != self.model.fingerprint():
                raise P.FingerprintMismatch("resume checkpoint fingerprint does not match model")
            v0 = resume.values
            iteration = resume.iteration
        else:
            v0 = self._initial_values()
            iteration = 0
        ring[0].copy_(torch.as_tensor(v0, dtype=torch.float64).to(self.dtype))
        order = [0]
        # Statistics of sweep i are read on the host one sweep late: sweep i+1
        # is already enqueued when the host waits for sweep i's (reduced)
        # statistics, so the device never idles on the host decision.  When
        # sweep i converged (or diverged), sweep i+1 was speculative: its
        # vector is dropped and V_i (another ring slot) is the result, so the
        # iteration count and values are exactly the eager loop's.
        pinned = self.device.type == "cuda"
        dstats = [torch.empty(4, dtype=torch.float64, device=self.device) for _ in range(2)]
        hstats = [torch.empty(4, dtype=torch.float64, pin_memory=pinned) for _ in range(2)]
        pending = None  # (iteration, want, event, host stats, order after the sweep)
        sweep_s = 0.0
        converged = False
        start = iteration
        ckpt = cfg.checkpoint_every > 0 and bool(cfg.checkpoint_path)
        fp = self.model.fingerprint()
        if ckpt and resume is None and self.rank == 0:
            P.save_checkpoint(cfg.checkpoint_path, ring[0].double().cpu().numpy(), iteration, fp)
        result_order = None
        ts = time.perf_counter()
        while True:
            stop = (iteration >= cfg.fixed_iterations if cfg.fixed_iterations > 0
                    else iteration >= start + cfg.max_iterations)
            launched = None
            if not stop:
                it = iteration + 1
                prev = order[-1]
                if len(order) < self.hist_cap:
                    nxt = len(order)
                else:
                    nxt = order.pop(0)
                want = cfg.fixed_iterations == 0 and len(order) + 1 >= self.hist_cap
                hist = [ring[k] for k in order] if (want and self.test == P.PERIODIC_SPAN) else []
                st = dstats[it & 1]
                if self._peer_slot(ring[nxt]) is not None and self.test != P.PERIODIC_SPAN:
                    self._peer_sweep(ring[prev], ring[nxt], self._peer_slot(ring[nxt]),
                                     self.test if want else None, st)
                else:
                    self._sweep(ring[prev], ring[nxt], None, self.test if want else None, hist, st)
                    self.reduce_stats(st)
                    self.refresh(ring[nxt])
                order.append(nxt)
                hs = hstats[it & 1]
                hs.copy_(st, non_blocking=pinned)
                ev = None
                if pinned:
                    ev = torch.cuda.Event()
                    ev.record()
                launched = (it, want, ev, hs, list(order))
                iteration = it
            if pending is not None:
                p_it, p_want, p_ev, p_hs, p_order = pending
                if p_ev is not None:
                    p_ev.synchronize()
                stv = p_hs.numpy()
                if stv[2] > NEG_INF:
                    bad = int(-stv[2])
                    raise P.NumericDivergence(f"non-finite value for state {bad} at iteration "
                                              f"{p_it}", p_it)
                done = False
                if p_want:
                    hi = stv[0]
                    lo = 0.0 if self.test == P.VALUE_SPAN else -stv[1]
                    done = bool(evaluate_test(self.test, float(hi), float(lo), cfg.epsilon, p_it))
                if ckpt and p_it % cfg.checkpoint_every == 0:
                    if self.plan is not None:
                        self.exchange(ring[p_order[-1]])  # a checkpoint holds all of V
                    if self.rank == 0:
                        P.save_checkpoint(cfg.checkpoint_path, ring[p_order[-1]].double().cpu().numpy(),
                                          p_it, fp)
                if done:
                    converged = True
                    iteration = p_it
                    result_order = p_order
                    break
            if launched is None:  # the iteration limit: the last launched sweep is the result
                converged = cfg.fixed_iterations > 0
                result_order = pending[4] if pending is not None else order
                break
            pending = launched
        sweep_s += time.perf_counter() - ts
        order = result_order
        vfinal = ring[order[-1]]
        actions = torch.zeros(n, dtype=torch.int32, device=self.device)
        self._sweep(vfinal, ring[order[0]] if len(order) > 1 else torch.empty_like(vfinal),
                    actions, None, [], None)
        self.exchange(actions, send=torch.empty(self.maxlen, dtype=torch.int32, device=self.device),
                      recv=torch.empty(self.maxlen * self.world, dtype=torch.int32,
                                       device=self.device))
        if self.plan is not None:
            self.exchange(vfinal)  # the result is the full value vector
        values = vfinal.double().cpu().numpy()
        policy = actions.cpu().numpy().astype(np.uint32)
        return ShardedResult(values, policy, iteration, converged, time.perf_counter() - t0,
                             sweep_s, self.bounds)

    def _initial_values(self) -> np.ndarray:
        if self.device.type == "cuda":
            return self.model.initial_values()
        from_fn = getattr(self.sweep, "initial_values", None)
        if from_fn is None:
            raise P.DeviceError("initial values need the device (or a sweep providing them)")
        return from_fn()
