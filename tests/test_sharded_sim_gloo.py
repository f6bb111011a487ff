"""Multi-rank simulation and simopt (sharded_sim.py)
under torch.distributed `gloo` on CPU, world sizes 2 and 3.

The per-rank simulation is the C oracle (oracle/pvi_oracle.c, the
reference's rollout restated) instead of the device kernel, so this runs the
driver code the GPU ranks run: candidate shards with the Evaluations
all-gathered, rollout shards (base_seed + first rollout) with the per-rollout
summaries all-gathered and reduced on the host in index order, and the
reference GA driven through pvi_simopt_config.score_batch on every rank.
Everything must equal the single-process evaluation bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from mp_util import collect


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_evaluate(preset):
    from oracle import cport

    def run(policies, n, seed, horizon, warmup):
        out = []
        for p in policies:
            if p.kind == 1:
                out.append(cport.eval_heuristic(preset, list(p.params), n, horizon, warmup, seed))
            else:
                out.append(cport.eval_table(preset, p.table, n, horizon, warmup, seed))
        return np.stack(out) if out else np.zeros((0, n, 7))
    return run


CANDS = {"a/m2/exp1": [[s] for s in range(11)],
         "b/m2/exp1": [[13, 12], [10, 10], [14, 9], [5, 20], [0, 0]],
         "c/m3/exp1": [[9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8],
                       [3, 4, 5, 6, 7, 2, 1, 10, 11, 12, 13, 14, 8, 9]]}


def _worker(rank, world, port, preset, n, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded_sim import ShardedEvaluator
        m = P.make_preset(preset)
        ev = ShardedEvaluator(m, evaluate=oracle_evaluate(preset))
        pols = [P.make_heuristic_policy(m, c) for c in CANDS[preset]]
        evs, summ = ev.evaluate(pols, P.RolloutConfig(n_rollouts=n, base_seed=42), per_rollout=True, mode=mode)
        out_q.put((rank, [(e.ret.mean, e.ret.sd, e.service_pct[0].mean, e.wastage_pct[0].sd,
                           e.holding_mean[e.products - 1].mean) for e in evs], summ))
    finally:
        dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for p in procs:
        p.start()
    outs = collect(procs, q, world, 600)
    return sorted(outs, key=lambda o: o[0])


@pytest.mark.parametrize("preset,world,n,mode", [("a/m2/exp1", 2, 300, "candidates"),
                                                 ("a/m2/exp1", 3, 301, "rollouts"),
                                                 ("b/m2/exp1", 2, 257, "rollouts"),
                                                 ("b/m2/exp1", 3, 200, "candidates"),
                                                 ("c/m3/exp1", 3, 150, "auto")])
def test_sharded_evaluation_bitwise(preset, world, n, mode):
    import paper_2303_10672_b200 as P
    m = P.make_preset(preset)
    summ = oracle_evaluate(preset)([P.make_heuristic_policy(m, c) for c in CANDS[preset]], n, 42, 365, 100)
    want = [(e.ret.mean, e.ret.sd, e.service_pct[0].mean, e.wastage_pct[0].sd,
             e.holding_mean[e.products - 1].mean) for e in P.sim_reduce(summ, m.products())]
    outs = _spawn(_worker, world, preset, n, mode)
    for rank, got, gsumm in outs:
        assert got == want, (rank, got, want)
        np.testing.assert_array_equal(gsumm, summ)


def _ga_worker(rank, world, port, preset, rollouts, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded_sim import ShardedEvaluator
        m = P.make_preset(preset)
        ev = ShardedEvaluator(m, evaluate=oracle_evaluate(preset))
        r = ev.simopt(rollouts_per_candidate=rollouts, base_seed=42, seed=1)
        out_q.put((rank, r.best, r.best_mean, r.generations, r.log))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("preset,world,rollouts", [("b/m2/exp1", 2, 64), ("a/m2/exp1", 3, 128)])
def test_sharded_simopt_same_trajectory(preset, world, rollouts):
    """The GA (b/m2) / grid (a/m2) with each batch sharded over the ranks
    follows exactly the single-process trajectory: same log, same best."""
    import paper_2303_10672_b200 as P
    from paper_2303_10672_b200.sharded_sim import ShardedEvaluator
    m = P.make_preset(preset)
    single = ShardedEvaluator(m, evaluate=oracle_evaluate(preset)).simopt(
        rollouts_per_candidate=rollouts, base_seed=42, seed=1)
    outs = _spawn(_ga_worker, world, preset, rollouts)
    for rank, best, mean, gens, log in outs:
        assert (best, mean, gens) == (single.best, single.best_mean, single.generations), rank
        assert log == single.log
