"""Multi-GPU policy simulation and simulation optimisation (SURVEY §8e,
BASELINE north_star: "simulation replicas and candidate parameters shard
trivially, with one final reduce").

One process per GPU under torch.distributed.  The reference fans out in two
places: evaluate_policy's rollouts (sim.hpp:145-170, chunks of 16 across
threads) and simopt's candidates (simopt.cpp:22-46, 65-83).  Here:

* candidate shards (a batch of >= world policies): rank r evaluates the
  contiguous policy range [p_r, p_{r+1}) with all rollouts on its GPU
  (pvi_sim_evaluate); the per-policy Evaluations (14 doubles each) are
  all-gathered.  Each Evaluation is computed exactly as on one GPU, so the
  result is bit-identical.
* rollout shards (fewer policies than ranks, e.g. cmd_evaluate of one VI
  policy over 10,000 rollouts): rank r simulates rollouts [f_r, f_{r+1}) of
  every policy.  Rollout i's RNG key is base_seed + i (rng.hpp:37-44), so
  the shard runs with base_seed + f_r; the per-rollout summaries are
  all-gathered, concatenated in rollout-index order and reduced on the host
  with detail::reduce's operations (pvi_sim_reduce) -- bit-identical to one
  device.  No ncclReduce for the means: it would change the summation order.

simopt: every rank runs the reference's serial GA / grid (same libstdc++
RNG, so the same trajectory) and each generation's batch is scored by the
sharded evaluator through pvi_simopt_config.score_batch: the collectives
of all ranks line up generation by generation.
"""
from __future__ import annotations

import time
from typing import Callable, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist

from . import pvi as P

# (policies, n_rollouts, base_seed, horizon_days, warmup_days) -> (n_pol, n, 7)
# per-rollout summaries: an injectable stand-in for the device kernel (tests
# run the C oracle here under gloo on CPU).
EvaluateFn = Callable[[Sequence[P.Policy], int, int, int, int], np.ndarray]


def balanced(n: int, parts: int) -> list:
    """Contiguous bounds of n items over `parts` shards (sizes differ by <= 1)."""
    q, r = divmod(n, parts)
    b = [0]
    for i in range(parts):
        b.append(b[-1] + q + (1 if i < r else 0))
    return b


def _pack(ev: P.Evaluation) -> list:
    out = [ev.ret.mean, ev.ret.sd]
    for k in range(2):
        out += [ev.service_pct[k].mean, ev.service_pct[k].sd, ev.wastage_pct[k].mean, ev.wastage_pct[k].sd,
                ev.holding_mean[k].mean, ev.holding_mean[k].sd]
    return out + [float(ev.products), float(ev.n_rollouts)]


def _unpack(v) -> P.Evaluation:
    v = [float(x) for x in v]
    K = P.KpiStat
    svc = [K(v[2], v[3]), K(v[8], v[9])]
    wst = [K(v[4], v[5]), K(v[10], v[11])]
    hld = [K(v[6], v[7]), K(v[12], v[13])]
    return P.Evaluation(K(v[0], v[1]), svc, wst, hld, int(v[14]), int(v[15]))


class ShardedEvaluator:
    """evaluate_policies / the simopt batch point over the ranks of `group`."""

    def __init__(self, model: P.Model, group=None, evaluate: Optional[EvaluateFn] = None,
                 comm_device: Optional[torch.device] = None):
        self.model = model
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.inject = evaluate
        if comm_device is None:
            backend = dist.get_backend(group) if dist.is_initialized() else "gloo"
            comm_device = (torch.device("cuda", torch.cuda.current_device()) if backend == "nccl"
                           else torch.device("cpu"))
        self.comm = comm_device
        self.products = model.products()
        self.device_seconds = 0.0  # this rank's time inside its own evaluations

    # -- local evaluation --------------------------------------------------
    def _local(self, policies, n, seed, cfg: P.RolloutConfig, per_rollout: bool):
        t0 = time.perf_counter()
        if self.inject is not None:
            summ = np.asarray(self.inject(policies, n, seed, cfg.horizon_days, cfg.warmup_days), np.float64)
            evs = P.sim_reduce(summ, self.products) if len(policies) else []
        else:
            c = P.RolloutConfig(horizon_days=cfg.horizon_days, warmup_days=cfg.warmup_days, n_rollouts=n,
                                base_seed=seed, device=cfg.device)
            evs, summ = P.evaluate_policies(self.model, policies, c, per_rollout=per_rollout)
        self.device_seconds += time.perf_counter() - t0
        return evs, summ

    def _all_gather_rows(self, rows: np.ndarray, counts: list) -> np.ndarray:
        """all-gather of per-rank row blocks (rows: count_r x k), padded to the
        largest count, concatenated in rank order."""
        k = rows.shape[1] if rows.ndim == 2 else 0
        mx = max(counts)
        buf = torch.zeros((mx, k), dtype=torch.float64, device=self.comm)
        if len(rows):
            buf[:len(rows)] = torch.from_numpy(np.ascontiguousarray(rows)).to(self.comm)
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        return np.concatenate([o[:c].cpu().numpy() for o, c in zip(outs, counts)], axis=0)

    # -- public ------------------------------------------------------------
    def evaluate(self, policies: Sequence[P.Policy], config: P.RolloutConfig, per_rollout: bool = False,
                 mode: str = "auto"):
        """(evaluations, summaries or None), identical on every rank and bit-identical
        to P.evaluate_policies on one device.  mode: auto | candidates | rollouts."""
        n_pol, n = len(policies), config.n_rollouts
        if n < 1:
            raise P.ParameterError("evaluation needs at least one rollout")
        if self.world == 1:
            return self._local(list(policies), n, config.base_seed, config, per_rollout)
        if mode == "auto":
            mode = "candidates" if n_pol >= self.world else "rollouts"
        if mode == "candidates":
            pb = balanced(n_pol, self.world)
            mine = list(policies[pb[self.rank]:pb[self.rank + 1]])
            evs, summ = self._local(mine, n, config.base_seed, config, per_rollout)
            counts = [pb[r + 1] - pb[r] for r in range(self.world)]
            packed = np.array([_pack(e) for e in evs], np.float64).reshape(len(mine), 16)
            allp = self._all_gather_rows(packed, counts)
            evals = [_unpack(row) for row in allp]
            summaries = None
            if per_rollout:
                loc = (np.asarray(summ, np.float64).reshape(len(mine), n * 7) if len(mine)
                       else np.zeros((0, n * 7)))
                summaries = self._all_gather_rows(loc, counts).reshape(n_pol, n, 7)
            return evals, summaries
        # rollout shards: [f_r, f_{r+1}) of every policy, RNG key base_seed + index
        rb = balanced(n, self.world)
        lo, hi = rb[self.rank], rb[self.rank + 1]
        counts = [rb[r + 1] - rb[r] for r in range(self.world)]
        if hi > lo:
            _, summ = self._local(list(policies), hi - lo, config.base_seed + lo, config, True)
            loc = np.asarray(summ, np.float64).transpose(1, 0, 2).reshape(hi - lo, n_pol * 7)
        else:
            loc = np.zeros((0, n_pol * 7))
        full = self._all_gather_rows(loc, counts).reshape(n, n_pol, 7).transpose(1, 0, 2)
        full = np.ascontiguousarray(full)
        return P.sim_reduce(full, self.products), (full if per_rollout else None)

    def score_batch(self, rollouts: int, base_seed: int, horizon_days: int = 365, warmup_days: int = 100):
        """The simopt batch point: candidates (n x dim ints) -> (means, sds)."""
        cfg = P.RolloutConfig(horizon_days=horizon_days, warmup_days=warmup_days, n_rollouts=rollouts,
                              base_seed=base_seed)

        def score(cands: np.ndarray):
            pols = [P.make_heuristic_policy(self.model, [int(x) for x in row]) for row in cands]
            evs, _ = self.evaluate(pols, cfg)
            return [e.ret.mean for e in evs], [e.ret.sd for e in evs]
        return score

    def simopt(self, rollouts_per_candidate: int = 4000, base_seed: int = 42, horizon_days: int = 365,
               warmup_days: int = 100, **kw) -> P.SimoptResult:
        """cmd_simopt's search with every batch sharded over the ranks; the
        same SimoptResult (trajectory, log, best) on every rank."""
        return P.simopt(self.model, rollouts_per_candidate=rollouts_per_candidate, base_seed=base_seed,
                        horizon_days=horizon_days, warmup_days=warmup_days,
                        score_batch=self.score_batch(rollouts_per_candidate, base_seed, horizon_days,
                                                     warmup_days), **kw)
