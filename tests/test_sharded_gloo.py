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
    it, conv, values, policy, bounds = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = cport.vi_solve(preset)
    assert (it, conv) == (want.iterations, want.converged)
    np.testing.assert_array_equal(values, want.values)
    np.testing.assert_array_equal(policy, want.policy)
    assert len(bounds) == world + 1 and bounds[-1] == len(values)
