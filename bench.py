#!/usr/bin/env python
"""Benchmark: Bellman evaluations per second of the B200 value-iteration
sweep (BASELINE.json metric), plus wall time to converge.

Workload (N=1 and every N): one synchronous Jacobi sweep of the >16M-state
scenario, Hendrix two-product b/m3/exp1 (16,777,216 states x 256 actions,
2.372e12 reference backup terms per sweep), f64, with the fused convergence
reduction.  A "step" is one full sweep over all states with V resident in
HBM; at N>1 each rank sweeps its cost-weighted state shard and the shards
are all-gathered over NCCL.  The sweep is the same at every N, so scaling
is "strong".  The unit of work is one reference backup term
(state, action, outcome) exactly as the reference enumerates it
(SURVEY §8d), so evals/s is comparable with the CPU reference arm.

  python bench.py [--gpus N --steps K --warmup W]            # our arm
  python bench.py --impl reference [--steps K --warmup W]     # reference CPU arm
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_TERM = {"f64": 8, "f32": 4}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="b/m3/exp1")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--algorithm", default="factored", choices=["exact", "factored"])
    ap.add_argument("--no-alt", action="store_true", help="skip timing the other algorithm")
    ap.add_argument("--no-simopt", action="store_true")
    ap.add_argument("--no-others", action="store_true", help="skip the a/m5 and c/m5 workloads")
    ap.add_argument("--no-ckpt-solve", action="store_true",
                    help="skip the second solve with the preset's checkpoint cadence")
    ap.add_argument("--no-solve", action="store_true", help="skip the time-to-converge solve")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of reference CPU work")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing


def init_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# work model (SURVEY §8d closed forms).  Built from the product model for our
# arm and from the reference library (oracle/_ref) alone for the reference
# arm, which must not load this repo's package.


class Work:
    """Reference backup terms (state, action, outcome) of a preset, per range."""

    def __init__(self, scenario: str, life: int, na: int, nb: int, states: int, actions: int,
                 terms: float):
        self.scenario, self.life, self.na, self.nb = scenario, life, na, nb
        self.states, self.actions, self.terms = states, actions, terms

    def range_terms(self, lo: int, hi: int) -> float:
        if self.scenario != "b":
            return self.terms * (hi - lo) / self.states
        m, na, nb = self.life, self.na, self.nb
        rem = np.arange(lo, hi, dtype=np.int64)
        ia = np.zeros(hi - lo, np.int64)
        ib = np.zeros(hi - lo, np.int64)
        for i, w in enumerate([na ** (m - 1 - k) * nb ** m for k in range(m)] +
                              [nb ** (m - 1 - k) for k in range(m)]):
            d = rem // w
            rem = rem % w
            if i < m:
                ia += d
            else:
                ib += d
        return float(np.sum((ia + 1) * (ib + 1), dtype=np.float64)) * self.actions

    def b_group(self) -> int:
        """States sharing the product-A digits (one contiguous block)."""
        return self.nb ** self.life


def work_from_model(model) -> Work:
    sc = model.scenario()
    life = model.state_arity() // 2 if sc == "b" else 0
    na = model.info.max_order_a + 1 if sc == "b" else 0
    nb = model.info.max_order_b + 1 if sc == "b" else 0
    return Work(sc, life, na, nb, model.state_count(), model.action_count(), model.terms_per_sweep())


def work_from_reference(preset: str) -> Work:
    """The same closed forms from the reference's own model (refbind), SURVEY §8d:
    A |S||A|(D+1) = |S||A||Omega|; C |S|(D+1)C(A_max+m, m) = |S||Omega|;
    B |A| sum_s (I_a+1)(I_b+1)."""
    from oracle import refbind as R
    c = R.counts(preset)
    sc = preset[0]
    if sc == "a":
        return Work("a", 0, 0, 0, c.states, c.actions, float(c.states) * c.actions * c.outcomes)
    if sc == "c":
        return Work("c", 0, 0, 0, c.states, c.actions, float(c.states) * c.outcomes)
    t = R.b_tables(preset)
    life = int(preset.split("/")[1][1:])
    na, nb = t["max_order_a"] + 1, t["max_order_b"] + 1
    per = lambda r: r ** life * (life * (r - 1) / 2.0 + 1.0)  # noqa: E731  sum over one product's digits of (I+1)
    return Work("b", life, na, nb, c.states, c.actions, float(c.actions) * per(na) * per(nb))


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md clocks line)


class Clocks:
    """SM clock and clock-event reasons sampled DURING the timed region.

    NVML in a thread every 10 ms (no process start-up: a 20-step headline
    region lasts ~0.1 s, shorter than nvidia-smi's first line); nvidia-smi
    -lms 200 only when NVML is unavailable."""
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines = []
        self.nv = None
        self.handle = None
        try:
            import pynvml
            pynvml.nvmlInit()
            try:  # the torch device's physical GPU (CUDA_VISIBLE_DEVICES may remap)
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.nv = pynvml
        except Exception:
            self.nv = None

    def start(self):
        self.samples, self.reason_bits = [], 0
        if self.nv is not None:
            self.stop_flag = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _poll(self):
        nv, h = self.nv, self.handle
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons",
                              getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
        while not self.stop_flag.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                if get_reasons is not None:
                    self.reason_bits |= int(get_reasons(h))
            except Exception:
                pass
            self.stop_flag.wait(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            nv = self.nv
            bits = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
                    "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
                    "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
                    "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}
            reasons = sorted(nm for nm, c in bits.items() if self.reason_bits & int(getattr(nv, c, 0)))
            try:
                smax = float(nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM))
            except Exception:
                smax = None
            return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                    "sm_max_mhz": smax, "reasons": reasons, "samples": len(self.samples),
                    "source": "nvml, 10 ms"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi -lms 200"}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference, compiled here)


def cpu_sample_plan(work: Work, budget_s: float, calib_rate: float):
    """Contiguous state ranges spread over the space, sized to ~budget_s of CPU work."""
    n = work.states
    group = work.b_group() if work.scenario == "b" else max(1, n // 4096)
    n_groups = max(1, n // group)
    per_group = work.terms / n_groups  # mean group size
    want = max(1, int(budget_s * calib_rate / max(per_group, 1.0)))
    want = min(want, n_groups)
    stride = max(1, n_groups // want)
    return [(g * group, min(n, (g + 1) * group)) for g in range(0, n_groups, stride)][:want]


def run_cpu_reference(work: Work, preset: str, precision: str, budget_s: float, V: np.ndarray,
                      offset: int = 0):
    """Time the reference's bellman_backup_batch (threads = all host cores) on a bounded
    sample; returns (terms/s, seconds, terms, description, threads)."""
    from oracle import refbind as R
    threads = os.cpu_count() or 1
    # calibrate with one small range
    plan = cpu_sample_plan(work, budget_s, 3e9)
    lo, hi = plan[len(plan) // 2]
    _, _, secs = R.backup_range(preset, V, lo, hi, f32=precision == "f32", threads=threads)
    rate = work.range_terms(lo, hi) / max(secs, 1e-6)
    plan = cpu_sample_plan(work, budget_s, rate)
    if offset:
        plan = plan[offset % len(plan):] + plan[:offset % len(plan)]
    terms = 0.0
    total = 0.0
    used = 0
    for lo, hi in plan:
        _, _, secs = R.backup_range(preset, V, lo, hi, f32=precision == "f32", threads=threads)
        total += secs
        terms += work.range_terms(lo, hi)
        used += hi - lo
        if total > budget_s * 1.5:
            break
    desc = (f"reference bellman_backup_batch over {used} of {work.states} states "
            f"({terms:.3e} terms, {100.0 * terms / work.terms:.2f}% of a sweep) in contiguous "
            f"tiles spread across the space")
    return terms / total, total, terms, desc, threads


# ---------------------------------------------------------------------------
# arms


def reference_arm(args, world, rank):
    """The reference's own CPU implementation (oracle/_ref = the unmodified
    reference sources) through its bellman_backup_batch, on all host cores.
    Nothing from this repo's package is loaded here.  One step = one bounded
    sample (~4 s) of the workload's sweep; value = terms/s over the samples."""
    from oracle import refbind as R
    if rank != 0:
        return
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libpvi_ref.so was not built (needs /root/reference)"}))
        return
    work = work_from_reference(args.workload)
    V = R.initial_values(args.workload)
    step_budget = 4.0
    rates, times, descs = [], [], []
    for k in range(args.warmup + args.steps):
        rate, secs, terms, desc, threads = run_cpu_reference(work, args.workload, args.precision,
                                                             step_budget, V, offset=k)
        if k >= args.warmup:
            rates.append(rate)
            times.append(secs)
            descs.append(desc)
    value = float(sum(r * t for r, t in zip(rates, times)) / sum(times))
    line = {
        "metric": "bellman_evals_per_sec", "value": value, "unit": "evals/s",
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "full_sweep_ms_extrapolated": 1e3 * work.terms / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic (deterministic preset tables; V = initial value)",
        "config": workload_config(work, args, world),
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads, "kind": "reference",
                         "sample": descs[0] + f"; one step = one ~{step_budget:.0f} s sample, "
                                              f"rotated through the space step by step"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def workload_config(work: Work, args, world):
    return {"workload": f"{args.workload} Bellman sweep ({work.states:,} states, "
                        f"{work.actions} actions, {args.precision})",
            "preset": args.workload, "states": work.states,
            "actions": work.actions, "terms_per_sweep": work.terms,
            "l2_flush": "256 MiB write between timed steps (V is 128 MiB, partials 2.4 GB)",
            "parallelism": f"state-shards x{world} (cost-weighted; per sweep the V runs each shard "
                           f"reads: NCCL all-to-all for factored B, all-gather otherwise)"}


def _load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def fp64_peak_tflops():
    """Measured FP64 FMA peak (tools/fp64_peak.cu on a B200, profiles/r2_fp64_peak.json),
    else the nominal 148 SMs x 64 FMA/clk x 2 x 1965 MHz."""
    j = _load_json("profiles/r2_fp64_peak.json")
    if j:
        best = max(r["tflops"] for r in j["results"] if r["kernel"] == "dfma")
        return best, "profiles/r2_fp64_peak.json (tools/fp64_peak.cu, DFMA, measured on a B200)"
    return 148 * 64 * 2 * 1.965e9 / 1e12, "nominal 148 SMs x 64 FMA/clk x 2 x 1965 MHz (no measurement)"


def essential_bytes(model, precision: str, states: int) -> float:
    """Bytes a sweep of `states` states cannot avoid moving: V in, V' and the
    argmax out, plus the per-state model table the kernel must read (factored
    B: ER / PT, 2 doubles per state)."""
    t = BYTES_PER_TERM[precision]
    per = 2 * t + 4
    if model.scenario() == "b" and getattr(model, "algorithm", "exact") == "factored":
        per += 16
    return float(per) * states


def compute_roofline(model, args, work, shard_terms, shard_states, kernel_ms, k_launches, step_ms):
    """The sweep is bound by the FP64 pipe, not by HBM: V and every table are
    L2-resident or staged in shared memory, and no stage is a dense contraction
    (no tensor-core form; B200's FP64 DMMA peak equals its FP64 FMA peak).
    `achieved` = the FP64 flops the kernels execute (factored: FMAs from the loop
    bounds, Model::factored_fmas; exact: the reference's 5 unfused ops per term)
    / the measured K1 time; `peak` = the measured DFMA peak.  `hbm` holds the
    memory side: the sweep's essential bytes and the ncu-measured DRAM traffic
    per sweep (profiles/k1_traffic.json)."""
    kernel_s = kernel_ms * 1e-3 / max(k_launches, 1)
    frac_of_sweep = shard_terms / work.terms
    if args.algorithm == "factored":
        flops = 2.0 * model.info.factored_fmas * frac_of_sweep
        flop_src = "2 x Model::factored_fmas (FMAs from the factored kernels' loop bounds)"
    else:
        flops = 5.0 * shard_terms
        flop_src = "5 unfused FP64 ops per reference term (the reference's expression)"
    peak, peak_src = fp64_peak_tflops()
    achieved = flops / kernel_s / 1e12 if kernel_ms else 0.0
    traffic = None
    for tj in _load_json("profiles/k1_traffic.json") or []:
        if (tj.get("workload"), tj.get("precision"), tj.get("algorithm")) == \
                (args.workload, args.precision, args.algorithm):
            traffic = tj.get("dram_bytes_per_launch")
            if traffic is not None:
                traffic *= frac_of_sweep
    peaks = _load_json("MEASURED_PEAKS.json") or {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    ess = essential_bytes(model, args.precision, shard_states)
    hbm = {"essential_bytes": ess,
           "achieved_gbs": ess / kernel_s / 1e9 if kernel_ms else 0.0, "peak": hbm_peak,
           "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
           "traffic_bytes": traffic}
    hbm["frac"] = hbm["achieved_gbs"] / hbm_peak
    if traffic:
        hbm["traffic_gbs"] = traffic / kernel_s / 1e9
        hbm["traffic_frac"] = hbm["traffic_gbs"] / hbm_peak
        hbm["traffic_over_essential"] = traffic / ess
    # the reference enumeration's gather bytes, for comparison only (L1/L2 hits)
    ref_terms = {"bytes_per_term": BYTES_PER_TERM[args.precision], "terms_per_launch": shard_terms,
                 "gbs": BYTES_PER_TERM[args.precision] * shard_terms / kernel_s / 1e9 if kernel_ms else 0.0,
                 "note": "one V[next] gather per reference term (SURVEY 8d); these are L1/L2 hits "
                         "or not performed at all by the factored kernels, so not a roofline"}
    return {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": "K1 launches of one sweep (factored B: k_b_fact_w16p + k_b_fact_qw4)",
            "flops_per_launch": flops, "flops_source": flop_src, "peak_source": peak_src,
            "kernel_ms_per_launch": kernel_ms / max(k_launches, 1),
            "kernel_share_of_step": kernel_ms / max(sum(step_ms), 1e-9),
            "hbm": hbm, "reference_term_gather": ref_terms}


def philox_peak():
    j = _load_json("profiles/r2_philox_peak.json")
    if not j:
        return None
    return max(r["gblocks_per_s"] for r in j["results"]) * 1e9


def simopt_section(P, world, rank, barrier):
    """Config 5: the GA on b/m2/exp1 (4096 rollouts per candidate), the
    exhaustive 21 x 21 grid, the optimality gap against the VI policy; with
    the rollout kernel's Philox blocks/s against the measured Philox peak."""
    import torch
    import torch.distributed as dist
    from paper_2303_10672_b200.sharded_sim import ShardedEvaluator
    mb = P.make_preset("b/m2/exp1")
    ev = ShardedEvaluator(mb)
    ev.simopt(rollouts_per_candidate=256, base_seed=42, seed=1, max_generations=2)  # warm-up
    ev.device_seconds = 0.0
    barrier()
    P.profile_enable(True)
    P.profile_sim_read()
    t0 = time.perf_counter()
    so = ev.simopt(rollouts_per_candidate=4096, base_seed=42, seed=1)
    wall = time.perf_counter() - t0
    blocks, days, kms = P.profile_sim_read()
    P.profile_enable(False)
    t = torch.tensor([wall, ev.device_seconds], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    wall_max, dev_max = float(t[0]), float(t[1])
    all_days = len(so.log) * 4096 * 465
    out = {"preset": "b/m2/exp1", "sampler": "ga", "best": so.best, "best_mean": so.best_mean,
           "generations": so.generations, "candidates": len(so.log), "n_gpus": world,
           "sharding": "candidates of each generation over the ranks" if world > 1 else "one device",
           "wall_seconds": wall_max, "device_seconds": dev_max,
           "rollout_days_per_s": all_days / max(dev_max, 1e-9)}
    peak = philox_peak()
    if kms > 0:
        out["k5_roofline"] = {
            "bound": "int (Philox4x32-10)", "philox_blocks_per_rollout_day": blocks / max(days, 1),
            "achieved_blocks_per_s": blocks / (kms * 1e-3), "kernel_ms": kms,
            "rollout_days_per_s_kernel": days / (kms * 1e-3),
            "peak_blocks_per_s": peak, "frac": (blocks / (kms * 1e-3) / peak) if peak else None,
            "peak_source": "profiles/r2_philox_peak.json (tools/philox_peak.cu on a B200)" if peak else None,
            "note": "rank-local counts: this rank's rollout kernels only"}
    if world == 1:
        ex = P.simopt(mb, sampler="exhaustive", rollouts_per_candidate=4096, base_seed=42)
        vi = P.run_value_iteration(mb, P.ViConfig())
        evs, _ = P.evaluate_policies(mb, [P.make_vi_policy(mb, vi.policy),
                                          P.make_heuristic_policy(mb, so.best),
                                          P.make_heuristic_policy(mb, ex.best)],
                                     P.RolloutConfig(n_rollouts=10_000, base_seed=42))
        vi_mean = evs[0].ret.mean
        out["exhaustive"] = {
            "candidates": len(ex.log), "best": ex.best, "best_mean": ex.best_mean,
            "device_seconds": ex.device_seconds,
            "rollout_days_per_s": len(ex.log) * 4096 * 465 / max(ex.device_seconds, 1e-9)}
        out["optimality_gap_pct"] = {
            "vi_policy_mean": vi_mean, "rollouts": 10_000,
            "ga_best": 100.0 * (vi_mean - evs[1].ret.mean) / abs(vi_mean),
            "exhaustive_best": 100.0 * (vi_mean - evs[2].ret.mean) / abs(vi_mean)}
    return out


OTHERS = ["a/m5/exp5", "c/m5/exp1", "c/m5/exp2"]


def other_workloads(P, args, barrier):
    """The other BASELINE configs: one factored f64 sweep (device events, L2
    flushed between steps), the solve to the reference's criterion, and the
    reference CPU solver on the host's cores (bounded sample) for each."""
    import torch
    out = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for preset in OTHERS:
        m = P.make_preset(preset).set_algorithm("factored")
        n = m.state_count()
        v = torch.as_tensor(np.random.default_rng(7).uniform(-5.0, 5.0, n), device="cuda")
        vn = torch.empty_like(v)
        stats = torch.empty(4, dtype=torch.float64, device="cuda")
        test = m.default_convergence_test()
        hist = [v.clone() for _ in range(6)] + [v] if test == P.PERIODIC_SPAN else []
        names = {0: "value_span", 1: "change_span", 2: "periodic_span"}
        st = torch.cuda.current_stream().cuda_stream

        def sweep():
            P.sweep_device(m, "f64", m.discount(), v.data_ptr(), vn.data_ptr(), None, 0, n, names[test],
                           [h.data_ptr() for h in hist], stats.data_ptr(), st)
        for _ in range(3):
            sweep()
        barrier()
        ms = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sweep()
            e1.record()
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        sweep_ms = statistics.median(ms)
        terms = m.terms_per_sweep()
        res = min((P.run_value_iteration(m) for _ in range(2)), key=lambda r: r.wall_seconds)
        entry = {"states": n, "terms_per_sweep": terms, "algorithm": "factored", "sweep_ms": sweep_ms,
                 "evals_per_s": terms / (sweep_ms * 1e-3), "solve_iterations": res.iterations,
                 "solve_wall_seconds": res.wall_seconds, "data": "V ~ U(-5, 5) seed 7 for the sweep"}
        if not args.no_cpu_baseline:
            from oracle import refbind as R
            if R.available():
                work = work_from_reference(preset)
                V = np.random.default_rng(7).uniform(-5.0, 5.0, n)
                rate, secs, sterms, desc, threads = run_cpu_reference(work, preset, "f64", 4.0, V)
                entry["cpu_baseline"] = {"value": rate, "unit": "evals/s", "cores": threads,
                                         "kind": "reference", "sample": desc, "seconds": secs,
                                         "extrapolated_solve_seconds": (res.iterations + 1) * terms / rate}
                entry["speedup_sweep"] = entry["evals_per_s"] / rate
                entry["speedup_solve"] = entry["cpu_baseline"]["extrapolated_solve_seconds"] / res.wall_seconds
        out[preset] = entry
    return out


def ours_arm(args, world, rank, local):
    import torch
    import torch.distributed as dist
    import paper_2303_10672_b200 as P
    from paper_2303_10672_b200.sharded import ShardedValueIteration

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model = P.make_preset(args.workload)
    n = model.state_count()
    cfg = P.ViConfig(precision=args.precision)
    dt = torch.float32 if args.precision == "f32" else torch.float64
    v0 = model.initial_values()
    vprev = torch.as_tensor(v0, device="cuda").to(dt)
    vnext = torch.empty_like(vprev)
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    test = model.default_convergence_test()
    # the periodic-span statistic (Scenario C) reads the 7 previous vectors
    hist = ([torch.empty_like(vprev).copy_(vprev) for _ in range(6)] + [vprev]
            if test == P.PERIODIC_SPAN else [])

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    exchange = os.environ.get("PVI_EXCHANGE", "peer")

    def timed(algorithm, steps, warmup, clocks=None):
        nonlocal vprev, vnext
        model.set_algorithm(algorithm)
        solver = ShardedValueIteration(model, cfg, exchange=exchange)
        bufs = solver.buffers()
        if bufs is not None:  # fused peer exchange: sweep into the IPC-shared replicas
            bufs[0].copy_(vprev)
            vprev, vnext = bufs
        for _ in range(warmup):
            solver.step(vprev, vnext, stats, test, hist)
        barrier()
        if clocks:
            clocks.start()
        P.profile_enable(True)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        barrier()
        for k in range(steps):
            flush.zero_()  # L2 flush between timed steps (outside the events)
            starts[k].record()
            solver.step(vprev, vnext, stats, test, hist)
            ends[k].record()
        barrier()
        kernel_ms, k_launches, all_launches = P.profile_read()
        P.profile_enable(False)
        clk = clocks.stop() if clocks else None
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        total = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(total, op=dist.ReduceOp.MAX)
        return solver, float(total.item()), step_ms, kernel_ms, k_launches, all_launches, clk

    clocks = Clocks(local)
    solver, total_ms, step_ms, kernel_ms, k_launches, all_launches, clk = timed(
        args.algorithm, args.steps, args.warmup, clocks)
    terms = model.terms_per_sweep()
    value = terms * args.steps / (total_ms * 1e-3)

    # roofline of the dominant kernels (the sweep's K1 launches: factored B =
    # k_b_fact_w16p + k_b_fact_qw4) on this rank's own states
    work = work_from_model(model)
    shard_terms = sum(work.range_terms(a, b) for a, b in solver.own_runs[solver.rank])
    shard_states = sum(b - a for a, b in solver.own_runs[solver.rank])
    roofline = compute_roofline(model, args, work, shard_terms, shard_states, kernel_ms, k_launches,
                                step_ms)
    if world > 1:
        roofline["exchange_bytes_per_rank"] = solver.read_set_bytes()
        roofline["exchange"] = ("fused peer stores from the sweep (NVLink, IPC)" if solver.buffers() is not None
                                else "NCCL all-to-all of the read set" if solver.plan is not None
                                else "NCCL all-gather")
        if solver.peer_error:
            roofline["peer_fallback"] = solver.peer_error
        roofline["shards"] = ("units: (x_3 pair, x_b column range) blocks" if solver.units is not None
                              else "contiguous state ranges")
    line = {"metric": "bellman_evals_per_sec", "value": value, "unit": "evals/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": args.precision,
            "data": "synthetic (deterministic preset tables; V = initial value)",
            "config": dict(workload_config(work, args, world), algorithm=args.algorithm),
            "clocks": clk, "gpu_launches": int(all_launches), "roofline": roofline}

    # the other algorithm on the same data (exact = bit-identical to the reference)
    if not args.no_alt:
        alt = "exact" if args.algorithm == "factored" else "factored"
        if model.scenario() in ("b", "c") or alt == "exact":
            _, t_alt, _, k_alt, kl_alt, _, _ = timed(alt, 2, 1)
            line["alternate"] = {"algorithm": alt, "ms_per_step": t_alt / 2,
                                 "value": terms * 2 / (t_alt * 1e-3), "unit": "evals/s",
                                 "kernel_ms_per_launch": k_alt / max(kl_alt, 1)}
        model.set_algorithm(args.algorithm)

    # e2e: the reference-facing call with HOST buffers, copies inside the timing
    if not args.no_e2e:
        # pinned host buffers, as a serving caller would hold them
        vh = torch.as_tensor(v0).to(dt).pin_memory().numpy()
        ov = torch.empty(solver.hi - solver.lo, dtype=dt).pin_memory().numpy()
        oa = torch.empty(solver.hi - solver.lo, dtype=torch.int32).pin_memory().numpy().view(np.uint32)
        P.bellman_backup_batch(model, vh, solver.lo, solver.hi, precision=args.precision,
                               out_values=ov, out_actions=oa)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            P.bellman_backup_batch(model, vh, solver.lo, solver.hi, precision=args.precision,
                                   out_values=ov, out_actions=oa)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        line["e2e"] = {"value": terms * args.steps / float(el.item()), "unit": "evals/s",
                       "h2d_bytes_per_step": int(vh.nbytes),
                       "d2h_bytes_per_step": int((solver.hi - solver.lo) * (vh.itemsize + 4)),
                       "call": "pvi_vi_backup (bellman_backup_batch) over the rank's shard, "
                               "host V in, host V' + argmax out"}

    # wall time to converge (the second half of the BASELINE metric)
    if not args.no_solve:
        barrier()
        runs, calls = [], []
        for _ in range(2):  # first call in the process pays allocations; report both
            t0 = time.perf_counter()
            if world == 1:  # the product API: pvi_vi_solve, V resident on the device throughout
                res = P.run_value_iteration(model, cfg)
                api = "pvi_vi_solve (run_value_iteration)"
            else:           # one process per GPU; the bench step's exchange per sweep
                sv = ShardedValueIteration(model, cfg, exchange=exchange)
                try:
                    res = sv.solve()
                finally:
                    sv.close()
                api = f"sharded.ShardedValueIteration (exchange={sv.exchange_mode})"
            calls.append(time.perf_counter() - t0)
            runs.append(res)
        best = min(range(2), key=lambda i: runs[i].wall_seconds)
        res = runs[best]
        line["solve"] = {"preset": args.workload, "iterations": res.iterations,
                         "converged": res.converged, "wall_seconds": res.wall_seconds,
                         "first_call_wall_seconds": runs[0].wall_seconds,
                         "python_call_seconds": calls[best],
                         "sweep_seconds": res.sweep_seconds, "algorithm": args.algorithm,
                         "api": api,
                         "checkpoints": "off (the reference cmd_solve writes one per sweep)"}
        if world == 1 and not args.no_ckpt_solve:
            import tempfile
            with tempfile.TemporaryDirectory() as tmp:
                every = model.preset_checkpoint_every or 1
                ck = P.ViConfig(precision=args.precision, checkpoint_every=every,
                                checkpoint_path=os.path.join(tmp, "checkpoint.ckpt"))
                rc = P.run_value_iteration(model, ck)
                line["solve"]["with_checkpoints"] = {
                    "checkpoint_every": every, "wall_seconds": rc.wall_seconds,
                    "writer": "async PVI1 (pinned double buffer + writer thread)"}

    # simulation optimisation (config 5): the reference GA on b/m2/exp1 with
    # 4096 rollouts per candidate, every generation scored in one device
    # batch; at N > 1 every generation's candidates are sharded over the ranks
    # (sharded_sim.ShardedEvaluator), timed as the max over ranks
    if not args.no_simopt:
        line_so = simopt_section(P, world, rank, barrier)
        if rank == 0:
            line["simopt"] = line_so

    # the other BASELINE configs, each against its own CPU baseline
    if rank == 0 and world == 1 and not args.no_others:
        line["other_workloads"] = other_workloads(P, args, barrier)

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import refbind as R
        if R.available():
            rate, secs, sterms, desc, threads = run_cpu_reference(work, args.workload,
                                                                  args.precision,
                                                                  args.cpu_budget, v0)
            line["cpu_baseline"] = {"value": rate, "unit": "evals/s", "cores": threads,
                                    "kind": "reference", "sample": desc,
                                    "seconds": secs}
            if "solve" in line:
                line["cpu_baseline"]["extrapolated_solve_seconds"] = (
                    line["solve"]["iterations"] + 1) * terms / rate
            if "simopt" in line:
                r = R.simopt("b/m2/exp1", rollouts=4096, eval_seed=42, ga_seed=1,
                             threads=threads)
                line["cpu_baseline"]["simopt_b_m2_exp1_seconds"] = r["wall"]
                line["simopt"]["cpu_wall_seconds"] = r["wall"]
                line["simopt"]["speedup_vs_cpu"] = r["wall"] / max(line["simopt"]["wall_seconds"], 1e-9)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    world, rank, local = init_dist()
    if args.impl == "reference":
        reference_arm(args, world, rank)
    else:
        ours_arm(args, world, rank, local)


if __name__ == "__main__":
    main()
