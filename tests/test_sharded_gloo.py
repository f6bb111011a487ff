"""Multi-rank host logic of the sharded value iteration under
torch.distributed `gloo`, world size 2 and 3, on CPU.

The per-shard sweep is the C oracle (oracle/pvi_oracle.c) instead of the
device kernel, so this exercises exactly the driver code the GPU ranks run:
cost-weighted partition, padded all-gather of V slices, MAX all-reduce of
(max, -min, first non-finite) statistics, the periodic-span history window,
the convergence decision and the policy all-gather.  The result must be
bit-identical to the single-process solve.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from mp_util import collect

NEG = -1.7976931348623157e308


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_sweep(preset, gamma):
    """A CPU stand-in for pvi_vi_sweep_device built on the C oracle."""
    from oracle import cport

    def sweep(vprev, vnext, actions, lo, hi, test, hist, stats):
        vals, acts = cport.backup_range(preset, vprev.numpy(), lo, hi)
        vnext[lo:hi] = torch.from_numpy(vals)
        if actions is not None:
            actions[lo:hi] = torch.from_numpy(acts.astype(np.int32))
        if stats is None:
            return
        cur = vals
        if not np.all(np.isfinite(cur)):
            bad = lo + int(np.argmin(np.isfinite(cur)))
            stats[2] = -float(bad)
        else:
            stats[2] = NEG
        if test is None or hi == lo:
            stats[0] = NEG
            stats[1] = NEG
            return
        if test == 2:  # periodic span (vi.hpp:136-156)
            h = [x[lo:hi].numpy() for x in hist] + [cur]
            acc = np.zeros(hi - lo)
            w = 1.0
            for j in range(7):
                acc = acc + w * (h[7 - j] - h[6 - j])
                w *= gamma
            st = acc
        else:
            d = cur - vprev[lo:hi].numpy()
            st = np.abs(d) if test == 0 else d
        stats[0] = float(st.max())
        stats[1] = float(-st.min())

    sweep.initial_values = lambda: cport.initial_values(preset)
    return sweep


def _worker(rank, world, port, preset, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded import ShardedValueIteration
        m = P.make_preset(preset)
        solver = ShardedValueIteration(m, P.ViConfig(), device=torch.device("cpu"),
                                       sweep=oracle_sweep(preset, m.discount()))
        res = solver.solve()
        if rank == 0:
            out_q.put((res.iterations, res.converged, res.values, res.policy, res.bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("preset,world", [("a/m2/exp1", 2), ("b/m2/exp1", 2), ("c/m3/exp1", 3)])
def test_sharded_solve_matches_single_process(preset, world):
    from oracle import cport
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, preset, q)) for r in range(world)]
    for p in procs:
        p.start()
    (it, conv, values, policy, bounds), = collect(procs, q, 1, 600)
    want = cport.vi_solve(preset)
    assert (it, conv) == (want.iterations, want.converged)
    np.testing.assert_array_equal(values, want.values)
    np.testing.assert_array_equal(policy, want.policy)
    assert len(bounds) == world + 1 and bounds[-1] == len(values)


# --- read-set exchange (factored Scenario B x_3-pair shards) ---------------

MOD = 1009.0


def _runs_checksum(v, runs):
    return float(sum(float(v[a:b].sum()) for a, b in runs))


def _fake_sweep(rank_runs):
    """A sweep that reads EVERY entry of its shard's read set: V'[s] =
    (3 V[s] + checksum(V over the read set) + s) mod 1009 (integer-valued
    doubles, so every sum is exact in any order)."""
    def sweep(vprev, vnext, actions, lo, hi, test, hist, stats):
        c = _runs_checksum(vprev, rank_runs(lo, hi))
        s = torch.arange(lo, hi, dtype=torch.float64)
        vnext[lo:hi] = torch.remainder(3.0 * vprev[lo:hi] + c + s, MOD)
        if stats is not None:
            stats[:] = torch.tensor([0.0, 0.0, NEG, 0.0], dtype=torch.float64)
    return sweep


def _rs_worker(rank, world, port, preset, steps, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded import ShardedValueIteration
        m = P.make_preset(preset).set_algorithm("factored")
        n = m.state_count()
        solver = ShardedValueIteration(m, P.ViConfig(), device=torch.device("cpu"),
                                       sweep=_fake_sweep(m.sweep_read_runs))
        assert solver.plan is not None
        v = torch.remainder(torch.arange(n, dtype=torch.float64) * 7.0, MOD)
        w = torch.empty_like(v)
        for _ in range(steps):
            solver.step(v, w)
            v, w = w, v
        runs = m.sweep_read_runs(solver.lo, solver.hi)
        mine = {(a, b): v[a:b].clone().numpy() for a, b in runs}
        received = solver.read_set_bytes()
        solver.exchange(v)  # full replica (what solve() returns)
        out_q.put((rank, runs, mine, v.numpy().copy(), received))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [3, 4])
def test_read_set_exchange_delivers_every_read(world):
    import paper_2303_10672_b200 as P
    preset, steps = "b/m3/exp1", 3
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    bounds = [int(b) for b in m.partition(world)]
    # single-process reference: every shard applies the rule on the global V
    v = torch.remainder(torch.arange(n, dtype=torch.float64) * 7.0, MOD)
    for _ in range(steps):
        w = v.clone()
        for r in range(world):
            lo, hi = bounds[r], bounds[r + 1]
            c = _runs_checksum(v, m.sweep_read_runs(lo, hi))
            w[lo:hi] = torch.remainder(3.0 * v[lo:hi] + c + torch.arange(lo, hi, dtype=torch.float64), MOD)
        v = w
    want = v.numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rs_worker, args=(r, world, port, preset, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = collect(procs, q, world, 600)
    for rank, runs, mine, full, received in got:
        for (a, b), vals in mine.items():
            np.testing.assert_array_equal(vals, want[a:b])
        np.testing.assert_array_equal(full, want)
        # the read set is a fraction of the all-gather's volume
        assert received < 0.5 * (n - (bounds[rank + 1] - bounds[rank])) * 8


def _fake_unit_sweep(model):
    """_fake_sweep over a unit shard: writes its own (pair, x_b range) runs
    from a checksum of its whole read set."""
    def sweep(vprev, vnext, actions, u_lo, u_hi, test, hist, stats):
        c = _runs_checksum(vprev, model.unit_runs(u_lo, u_hi, read=True))
        for a, b in model.unit_runs(u_lo, u_hi):
            s = torch.arange(a, b, dtype=torch.float64)
            vnext[a:b] = torch.remainder(3.0 * vprev[a:b] + c + s, MOD)
        if stats is not None:
            stats[:] = torch.tensor([0.0, 0.0, NEG, 0.0], dtype=torch.float64)
    return sweep


def _unit_worker(rank, world, port, preset, steps, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded import ShardedValueIteration
        m = P.make_preset(preset).set_algorithm("factored")
        n = m.state_count()
        solver = ShardedValueIteration(m, P.ViConfig(), device=torch.device("cpu"),
                                       sweep=_fake_unit_sweep(m), shards="units")
        assert solver.units is not None and solver.plan is not None
        v = torch.remainder(torch.arange(n, dtype=torch.float64) * 7.0, MOD)
        w = torch.empty_like(v)
        for _ in range(steps):
            solver.step(v, w)
            v, w = w, v
        ub = solver.units
        runs = m.unit_runs(ub[rank], ub[rank + 1], read=True)
        mine = {(a, b): v[a:b].clone().numpy() for a, b in runs}
        solver.exchange(v)
        out_q.put((rank, mine, v.numpy().copy(), solver.read_set_bytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [3, 4])
def test_unit_shard_exchange_delivers_every_read(world):
    import paper_2303_10672_b200 as P
    preset, steps = "b/m3/exp1", 2
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    ub = [int(b) for b in m.unit_partition(world)]
    v = torch.remainder(torch.arange(n, dtype=torch.float64) * 7.0, MOD)
    for _ in range(steps):
        w = v.clone()
        for r in range(world):
            c = _runs_checksum(v, m.unit_runs(ub[r], ub[r + 1], read=True))
            for a, b in m.unit_runs(ub[r], ub[r + 1]):
                w[a:b] = torch.remainder(3.0 * v[a:b] + c + torch.arange(a, b, dtype=torch.float64), MOD)
        v = w
    want = v.numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_unit_worker, args=(r, world, port, preset, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = collect(procs, q, world, 900)
    for rank, mine, full, received in got:
        for (a, b), vals in mine.items():
            np.testing.assert_array_equal(vals, want[a:b])
        np.testing.assert_array_equal(full, want)
        assert 0 < received < 0.6 * n * 8


# --- fused peer exchange setup: all ranks agree ------------------------------

def _peer_setup_worker(rank, world, port, fail_rank, fail_where, out_q):
    """_setup_peers with the device calls stubbed: one rank cannot allocate
    or map; every rank must fall back to the read-set exchange together."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200 import sharded as S

        class FakeBuf:
            def __init__(self, count, dtype):
                if rank == fail_rank and fail_where == "alloc":
                    raise P.DeviceError("cudaMalloc failed (stub)")

            def ipc_handle(self):
                return bytes([rank]) * 64

        opened, closed = [], []

        def fake_open(h):
            if rank == fail_rank and fail_where == "open":
                raise P.DeviceError("peer access unavailable (stub)")
            opened.append(h[0])
            return 1000 + h[0]

        S.P.DeviceBuffer = FakeBuf
        S.P.ipc_open = fake_open
        S.P.ipc_close = lambda ptr: closed.append(ptr)
        m = P.make_preset("b/m2/exp1").set_algorithm("factored")
        solver = S.ShardedValueIteration(m, P.ViConfig(), device=torch.device("cpu"),
                                         sweep=_fake_sweep(m.sweep_read_runs))
        solver._setup_peers()
        out_q.put((rank, solver.peer is None, solver.exchange_mode, solver.peer_error,
                   sorted(opened), sorted(closed)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_where", ["alloc", "open"])
def test_peer_setup_falls_back_on_every_rank(fail_where):
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_setup_worker, args=(r, world, port, 1, fail_where, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(collect(procs, q, world, 600))
    for rank, no_peer, mode, why, opened, closed in res:
        assert no_peer and mode == "runs" and why, (rank, no_peer, mode, why)
        # whatever a healthy rank mapped before the vote is unmapped again
        assert [1000 + q for q in opened] == closed
    if fail_where == "open":  # the healthy ranks had mapped both peers' two buffers
        assert [len(r[4]) for r in res] == [4, 0, 4]
