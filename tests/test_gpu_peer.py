"""Fused exchange over peer memory (pvi_vi_sweep_device_peers): the
factored B stage-2 finalize stores each V' entry into the replica of every
peer whose next sweep reads it.

One GPU here, so the peers are (1) other buffers of the same process and
(2) a second process on the same GPU mapping this one's buffer through CUDA
IPC (ranks synchronised with gloo on the host; no kernel waits on another
process).  Both check: the peer replica holds exactly this shard's V' on the
peer's read set (pvi_sweep_read_runs) and nothing elsewhere."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from mp_util import collect

pytestmark = pytest.mark.gpu


def _covered(runs, lo, hi, n):
    mask = np.zeros(n, bool)
    for a, b in runs:
        mask[max(a, lo):min(b, hi)] = True
    return mask


def test_peer_stores_in_process(pvi):
    m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
    n = m.state_count()
    b = [int(x) for x in m.partition(8)]
    V = np.random.default_rng(6).uniform(-20.0, 20.0, n)
    full, _ = pvi.bellman_backup_batch(m, V, 0, n)
    vprev = torch.as_tensor(V, device="cuda")
    r = 3
    lo, hi = b[r], b[r + 1]
    vnext = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    peers = {q: pvi.DeviceBuffer(n) for q in (1, 6, 7)}
    tens = {q: torch.as_tensor(buf, device="cuda") for q, buf in peers.items()}
    for t in tens.values():
        t.fill_(float("nan"))
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    pvi.sweep_device_peers(m, "f64", m.discount(), vprev.data_ptr(), vnext.data_ptr(), lo, hi,
                           [(peers[q].ptr, b[q], b[q + 1]) for q in peers], test="change_span",
                           stats_ptr=stats.data_ptr(), stream_ptr=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(vnext[lo:hi].cpu().numpy(), full[lo:hi])
    for q, t in tens.items():
        got = t.cpu().numpy()
        want_mask = _covered(m.sweep_read_runs(b[q], b[q + 1]), lo, hi, n)
        assert want_mask.any()
        np.testing.assert_array_equal(got[want_mask], full[want_mask])
        assert np.isnan(got[~want_mask]).all()  # nothing outside the peer's read set
    # the same sweep without peers: identical values and statistics
    vnext2 = torch.empty_like(vnext)
    stats2 = torch.empty_like(stats)
    pvi.sweep_device(m, "f64", m.discount(), vprev.data_ptr(), vnext2.data_ptr(), None, lo, hi,
                     "change_span", (), stats2.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(vnext2[lo:hi], vnext[lo:hi]) and torch.equal(stats2, stats)


@pytest.mark.parametrize("preset,algo,test", [("b/m3/exp4", "exact", "change_span"),
                                               ("a/m5/exp5", "factored", "value_span"),
                                               ("c/m5/exp1", "factored", "change_span"),
                                               ("a/m3/exp6", "exact", "value_span")])
def test_peer_broadcast_for_whole_v_sweeps(pvi, preset, algo, test):
    """Every sweep but factored B's gathers from all of V: its finalize
    broadcasts each V' entry of [lo, hi) into every peer replica (and
    nothing else), with the same values and statistics as without peers."""
    m = pvi.make_preset(preset).set_algorithm(algo)
    n = m.state_count()
    b = [int(x) for x in m.partition(4)]
    V = np.random.default_rng(12).uniform(-20.0, 20.0, n)
    vprev = torch.as_tensor(V, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    r = 1
    lo, hi = b[r], b[r + 1]
    peers = {q: pvi.DeviceBuffer(n) for q in (0, 2, 3)}
    tens = {q: torch.as_tensor(buf, device="cuda") for q, buf in peers.items()}
    for t in tens.values():
        t.fill_(float("nan"))
    vnext = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    pvi.sweep_device_peers(m, "f64", m.discount(), vprev.data_ptr(), vnext.data_ptr(), lo, hi,
                           [(peers[q].ptr, b[q], b[q + 1]) for q in peers], test=test,
                           stats_ptr=stats.data_ptr(), stream_ptr=st)
    vnext2 = torch.full_like(vnext, float("nan"))
    stats2 = torch.empty_like(stats)
    pvi.sweep_device(m, "f64", m.discount(), vprev.data_ptr(), vnext2.data_ptr(), None, lo, hi, test, (),
                     stats2.data_ptr(), st)
    torch.cuda.synchronize()
    assert torch.equal(vnext[lo:hi], vnext2[lo:hi]) and torch.equal(stats, stats2)
    want = vnext2[lo:hi].cpu().numpy()
    for q, t in tens.items():
        got = t.cpu().numpy()
        np.testing.assert_array_equal(got[lo:hi], want)
        assert np.isnan(got[:lo]).all() and np.isnan(got[hi:]).all()


def test_peer_sweep_refuses_periodic_span(pvi):
    m = pvi.make_preset("c/m3/exp1")
    v = torch.zeros(m.state_count(), dtype=torch.float64, device="cuda")
    with pytest.raises(pvi.ParameterError):
        pvi.sweep_device_peers(m, "f64", m.discount(), v.data_ptr(), v.data_ptr(), 0, 10, [],
                               test="periodic_span")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2303_10672_b200 as pvi
        m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
        n = m.state_count()
        b = [int(x) for x in m.partition(world)]
        lo, hi = b[rank], b[rank + 1]
        V = np.random.default_rng(6).uniform(-20.0, 20.0, n)
        mine = pvi.DeviceBuffer(n)
        tmine = torch.as_tensor(mine, device="cuda")
        tmine.fill_(float("nan"))
        torch.cuda.synchronize()
        handles = [None] * world
        dist.all_gather_object(handles, mine.ipc_handle())
        peers = []
        for p in range(world):
            if p != rank:
                peers.append((pvi.ipc_open(handles[p]), b[p], b[p + 1]))
        vprev = torch.as_tensor(V, device="cuda")
        pvi.sweep_device_peers(m, "f64", m.discount(), vprev.data_ptr(), tmine.data_ptr(), lo, hi, peers,
                               stream_ptr=torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        dist.barrier()  # every rank's sweep (and its stores into the others) is done
        got = tmine.cpu().numpy()
        full, _ = pvi.bellman_backup_batch(m, V, 0, n)
        own = np.zeros(n, bool)
        own[lo:hi] = True
        runs = m.sweep_read_runs(lo, hi)
        need = np.zeros(n, bool)
        for a, bb in runs:
            need[a:bb] = True
        ok_own = bool(np.array_equal(got[own], full[own]))
        from_peers = need & ~own
        ok_peer = bool(np.array_equal(got[from_peers], full[from_peers]))
        untouched = bool(np.isnan(got[~(own | need)]).all())
        dist.barrier()
        for p in peers:
            pvi.ipc_close(p[0])
        q.put((rank, ok_own, ok_peer, untouched, int(from_peers.sum())))
    finally:
        dist.destroy_process_group()


def test_peer_stores_across_processes_ipc():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = collect(procs, q, world, 600)
    for rank, ok_own, ok_peer, untouched, n_from_peers in res:
        assert n_from_peers > 0
        assert ok_own and ok_peer and untouched, (rank, ok_own, ok_peer, untouched)


def _solve_worker(rank, world, port, preset, algo, exchange, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2303_10672_b200 as pvi
        from paper_2303_10672_b200.sharded import ShardedValueIteration
        m = pvi.make_preset(preset).set_algorithm(algo)
        solver = ShardedValueIteration(m, pvi.ViConfig(), exchange=exchange)
        if exchange == "peer":
            assert solver.buffers() is not None
        res = solver.solve()
        solver.close()
        if rank == 0:
            q.put((res.iterations, res.converged, res.values, res.policy, solver.read_set_bytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("preset,algo,exchange,world", [("b/m3/exp1", "factored", "peer", 2),
                                                        ("a/m2/exp1", "factored", "peer", 2),
                                                        ("b/m2/exp1", "exact", "peer", 3),
                                                        ("c/m5/exp2", "factored", "runs", 2),
                                                        ("c/m3/exp1", "factored", "runs", 3)])
def test_sharded_solve_multi_process(pvi, preset, algo, exchange, world):
    """The whole sharded solve, ranks as processes on this one GPU (gloo for
    the statistics; no kernel waits on another rank): the fused peer stores
    (factored B: to the readers; other sweeps: broadcast into full replicas)
    and the weekday shards of factored C (read set: one next-weekday slice,
    all-to-all) give the same iterations, values and policy as the
    single-process solve.  The host reads each sweep's statistics one sweep
    late (speculative next sweep), which must not change the result."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, preset, algo, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    (it, conv, values, policy, rbytes), = collect(procs, q, 1, 900)
    want = pvi.run_value_iteration(pvi.make_preset(preset).set_algorithm(algo))
    assert (it, conv) == (want.iterations, want.converged)
    np.testing.assert_array_equal(values, want.values)
    np.testing.assert_array_equal(policy, want.policy)
    if preset.startswith("c/"):
        n = len(values)
        assert rbytes <= 8 * (n // 7) * 3  # a weekday shard refreshes ~one weekday slice


# --- unit shards: (x_3 pair, x_b column range) blocks ------------------------

@pytest.mark.parametrize("parts", [8, 5, 3])
def test_unit_shards_equal_full_sweep(pvi, parts):
    """Every rank's unit-shard sweep (a few (pair, x_b range) segments) is
    bit-identical to its states of one full sweep, reads only its read
    runs (all else NaN), and the shards' statistics combine to the full
    sweep's."""
    m = pvi.make_preset("b/m3/exp1").set_algorithm("factored")
    n = m.state_count()
    V = np.random.default_rng(9).uniform(-20.0, 20.0, n)
    vprev = torch.as_tensor(V, device="cuda")
    full = torch.empty_like(vprev)
    fst = torch.empty(4, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    pvi.sweep_device(m, "f64", m.discount(), vprev.data_ptr(), full.data_ptr(), None, 0, n, "change_span",
                     (), fst.data_ptr(), st)
    b = [int(x) for x in m.unit_partition(parts)]
    assert b[0] == 0 and b[-1] == m.unit_count() and len(set(b)) == parts + 1
    covered = np.zeros(n, np.int32)
    agg = np.array([-np.inf, -np.inf, -np.inf])
    for r in range(parts):
        own = m.unit_runs(b[r], b[r + 1])
        rd = m.unit_runs(b[r], b[r + 1], read=True)
        Vp = torch.full_like(vprev, float("nan"))
        for x, y in rd:
            Vp[x:y] = vprev[x:y]
        out = torch.full_like(vprev, float("nan"))
        sts = torch.empty(4, dtype=torch.float64, device="cuda")
        pvi.sweep_device_units(m, m.discount(), Vp.data_ptr(), out.data_ptr(), b[r], b[r + 1],
                               test="change_span", stats_ptr=sts.data_ptr(), stream_ptr=st)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        f = full.cpu().numpy()
        mask = np.zeros(n, bool)
        for x, y in own:
            mask[x:y] = True
        covered += mask
        np.testing.assert_array_equal(o[mask], f[mask])
        assert np.isnan(o[~mask]).all()
        agg = np.maximum(agg, sts.cpu().numpy()[:3])
    assert (covered == 1).all()  # the shards tile the state space
    np.testing.assert_array_equal(agg, fst.cpu().numpy()[:3])


@pytest.mark.parametrize("preset,algo,exchange", [("b/m3/exp1", "factored", "peer"),
                                                  ("c/m5/exp1", "factored", "runs"),
                                                  ("b/m3/exp4", "exact", "peer")])
def test_eight_rank_solve_on_one_gpu(pvi, preset, algo, exchange):
    """The 8-rank layouts the bench would use on an 8-GPU node, as 8
    processes sharing this GPU: b/m3/exp1 unit shards with fused peer stores,
    c/m5/exp1 weekday shards (7 weekdays over 8 ranks: one rank owns no
    state), b/m3/exp4 exact with broadcast peer stores.  Same iterations,
    values and policy as one process."""
    world = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, preset, algo, exchange, q))
             for r in range(world)]
    for p in procs:
        p.start()
    (it, conv, values, policy, _), = collect(procs, q, 1, 1500)
    want = pvi.run_value_iteration(pvi.make_preset(preset).set_algorithm(algo))
    assert (it, conv) == (want.iterations, want.converged)
    np.testing.assert_array_equal(values, want.values)
    np.testing.assert_array_equal(policy, want.policy)
