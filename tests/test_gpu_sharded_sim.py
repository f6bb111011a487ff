"""Sharded simulation on the device (sharded_sim.py): two ranks on this
box's one GPU (gloo carries the all-gathers; no kernel waits on another
rank), each running pvi_sim_evaluate on its candidate or rollout shard.
Must equal the single-process device evaluation bit for bit, and the
sharded GA must follow the reference's cmd_simopt trajectory (SURVEY App. B:
b/m2/exp1 best (13, 12), 7 generations, 329 candidates)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from mp_util import collect

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "simopt_golden.npz"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, job, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_10672_b200 as P
        from paper_2303_10672_b200.sharded_sim import ShardedEvaluator
        if job == "simopt":
            m = P.make_preset("b/m2/exp1")
            r = ShardedEvaluator(m).simopt(rollouts_per_candidate=4096, base_seed=42, seed=1)
            out_q.put((rank, r.best, r.best_mean, r.generations, [(g, v, mu, sd) for g, v, mu, sd in r.log]))
        else:
            preset, mode = job
            m = P.make_preset(preset)
            if mode == "vi":
                res = P.run_value_iteration(m)
                pols = [P.make_vi_policy(m, res.policy)]
                n = 10_000
            else:
                pols = [P.make_heuristic_policy(m, [s]) for s in range(11)]
                n = 4096
            evs, summ = ShardedEvaluator(m).evaluate(pols, P.RolloutConfig(n_rollouts=n, base_seed=42),
                                                     per_rollout=True, mode=mode if mode != "vi" else "auto")
            out_q.put((rank, [(e.ret.mean, e.ret.sd, e.service_pct[0].mean, e.wastage_pct[0].sd) for e in evs],
                       summ))
    finally:
        dist.destroy_process_group()


def _spawn(world, job):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = collect(procs, q, world, 900)
    return outs


@pytest.mark.parametrize("job", [("a/m2/exp1", "candidates"), ("a/m2/exp1", "rollouts"),
                                 ("b/m2/exp1", "vi")])
def test_sharded_device_evaluation_bitwise(pvi, job):
    preset, mode = job
    m = pvi.make_preset(preset)
    if mode == "vi":
        pols = [pvi.make_vi_policy(m, pvi.run_value_iteration(m).policy)]
        n = 10_000
    else:
        pols = [pvi.make_heuristic_policy(m, [s]) for s in range(11)]
        n = 4096
    evs, summ = pvi.evaluate_policies(m, pols, pvi.RolloutConfig(n_rollouts=n, base_seed=42), per_rollout=True)
    want = [(e.ret.mean, e.ret.sd, e.service_pct[0].mean, e.wastage_pct[0].sd) for e in evs]
    for rank, got, gsumm in _spawn(2, job):
        assert got == want, rank
        np.testing.assert_array_equal(gsumm, summ)


def test_sharded_device_ga_matches_reference_trajectory():
    outs = _spawn(2, "simopt")
    log = GOLD["simopt|b/m2/exp1|log_values"]
    scores = GOLD["simopt|b/m2/exp1|log_scores"]
    for rank, best, mean, gens, got_log in outs:
        assert best == [13, 12] and gens == 7 and len(got_log) == 329
        assert mean == float(GOLD["simopt|b/m2/exp1|score"][0])
        assert [v for _, v, _, _ in got_log] == log.tolist()
        assert [[g, mu, sd] for g, _, mu, sd in got_log] == scores.tolist()
