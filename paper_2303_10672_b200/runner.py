"""cmd_solve / cmd_simopt / cmd_evaluate (proj/src/runner.cpp:303-480) over
the B200 engine, writing the reference's output files byte for byte (except
the wall-clock and thread-count report lines): checkpoint.ckpt (PVI1),
policy.csv + policy.csv.meta.json, report.txt, search_log.csv,
best_params.txt, kpis.csv.  Formats follow proj/src/io.cpp (RFC-4180 CSV,
17-significant-digit doubles) and runner.cpp:38-300.

This is host plumbing around the hot path; all compute goes
through the C ABI.
"""
from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import pvi as P


# ---------------------------------------------------------------------------
# io.cpp


def format_double(v: float) -> str:
    """std::ostream with precision 17 (io.cpp:93-98)."""
    return "%.17g" % v


def csv_field(raw: str) -> str:
    if not any(c in raw for c in ',"\n\r'):
        return raw
    return '"' + raw.replace('"', '""') + '"'


def csv_row(fields) -> str:
    return ",".join(csv_field(str(f)) for f in fields) + "\n"


def atomic_write_text(path: str, text) -> None:
    """Temp file + rename (io.cpp atomic_write_text); text is str or bytes."""
    tmp = path + ".tmp"
    try:
        if isinstance(text, (bytes, bytearray, memoryview)):
            with open(tmp, "wb") as f:
                f.write(text)
        else:
            with open(tmp, "w", newline="") as f:
                f.write(text)
        os.replace(tmp, path)
    except OSError as e:
        raise P.IoError(f"cannot write {path}: {e}") from e


def parse_csv(text: str):
    rows, row, field, quoted, i = [], [], [], False, 0
    while i < len(text):
        c = text[i]
        if quoted:
            if c == '"':
                if i + 1 < len(text) and text[i + 1] == '"':
                    field.append('"')
                    i += 1
                else:
                    quoted = False
            else:
                field.append(c)
        elif c == '"':
            quoted = True
        elif c == ",":
            row.append("".join(field))
            field = []
        elif c == "\n":
            row.append("".join(field))
            field = []
            rows.append(row)
            row = []
        elif c != "\r":
            field.append(c)
        i += 1
    if field or row:
        row.append("".join(field))
        rows.append(row)
    return rows


# ---------------------------------------------------------------------------
# column naming (runner.cpp:38-88)


def state_column_names(model: P.Model):
    sc = model.scenario()
    if sc == "a":
        m, lead = _a_life_lead(model)
        return [f"transit_{k}" for k in range(lead - 1, 0, -1)] + \
               [f"stock_{j}" for j in range(m, 0, -1)]
    if sc == "b":
        m = model.state_arity() // 2
        return [f"a_stock_{j}" for j in range(m, 0, -1)] + [f"b_stock_{j}" for j in range(m, 0, -1)]
    m = model.state_arity()
    return ["weekday"] + [f"stock_{j}" for j in range(m - 1, 0, -1)]


def _a_life_lead(model: P.Model):
    mat = model.fingerprint_material()
    kv = dict(x.split("=", 1) for x in mat.split(";"))
    return int(kv["m"]), int(kv["L"])


def action_column_names(model: P.Model):
    return ["order_a", "order_b"] if model.scenario() == "b" else ["order"]


def heuristic_kind(model: P.Model) -> str:
    return {"a": "base_stock", "b": "modified_base_stock", "c": "weekday_sS"}[model.scenario()]


def report_text(name: str, scenario: str, threads: int, extra) -> str:
    lines = [f"name = {name}", f"scenario = {scenario}", f"threads = {threads}"]
    lines += [f"{k} = {v}" for k, v in extra]
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# policy CSV (runner.cpp:90-166)


def policy_to_csv(model: P.Model, actions: np.ndarray) -> bytes:
    """runner.cpp:90-107: the header row, then one row per state formatted
    on the device (pvi_policy_csv_format)."""
    header = csv_row(state_column_names(model) + action_column_names(model))
    return header.encode() + model.policy_csv_body(actions)


def write_policy_outputs(model: P.Model, actions: np.ndarray, scenario: str, name: str,
                         csv_path: str) -> None:
    atomic_write_text(csv_path, policy_to_csv(model, actions))
    meta = {"scenario": scenario, "name": name, "fingerprint": model.fingerprint().hex(),
            "states": model.state_count()}
    atomic_write_text(csv_path + ".meta.json", json.dumps(meta, indent=2, sort_keys=True) + "\n")


def policy_from_csv(model: P.Model, csv_path: str) -> np.ndarray:
    if not os.path.exists(csv_path):
        raise P.IoError(f"cannot open policy CSV: {csv_path}")
    meta_path = csv_path + ".meta.json"
    try:
        meta = json.loads(open(meta_path).read())
    except (OSError, ValueError) as e:
        raise P.FormatError(f"cannot parse policy metadata {meta_path}: {e}") from e
    fp = model.fingerprint().hex()
    if meta.get("fingerprint", "") != fp:
        raise P.FingerprintMismatch(f"policy fingerprint {meta.get('fingerprint', '')} does not "
                                    f"match the configured scenario's {fp}")
    try:
        text = open(csv_path, "rb").read()
    except OSError as e:
        raise P.IoError(f"cannot read {csv_path}: {e}") from e
    return model.policy_from_csv_text(text)  # parsed on the device (pvi_policy_csv_parse)


# ---------------------------------------------------------------------------
# commands


@dataclass
class SolveOutcome:
    states: int
    iterations: int
    converged: bool
    wall_seconds: float
    policy_csv: str
    checkpoint: str
    report: str


def cmd_solve(preset: str, output_dir: str, resume: bool = False, threads: Optional[int] = None,
              config: Optional[P.ViConfig] = None, algorithm: str = "exact") -> SolveOutcome:
    """runner.cpp:303-350."""
    t0 = time.perf_counter()
    threads = threads or os.cpu_count() or 1
    os.makedirs(output_dir, exist_ok=True)
    ckpt = os.path.join(output_dir, "checkpoint.ckpt")
    policy_csv = os.path.join(output_dir, "policy.csv")
    report = os.path.join(output_dir, "report.txt")
    model = P.make_preset(preset).set_algorithm(algorithm)
    cfg = config or P.ViConfig()
    if cfg.checkpoint_every == 0:
        cfg.checkpoint_every = model.preset_checkpoint_every or (100 if model.scenario() == "a" else 1)
    if cfg.fixed_iterations == 0 and model.preset_fixed_iterations:
        cfg.fixed_iterations = model.preset_fixed_iterations
    cfg.checkpoint_path = ckpt
    res_from = P.load_checkpoint(ckpt, model.fingerprint()) if resume else None
    res = P.run_value_iteration(model, cfg, res_from)
    P.save_checkpoint(ckpt, res.values, res.iterations, res.fingerprint)
    write_policy_outputs(model, res.policy, model.scenario(), preset, policy_csv)
    wall = time.perf_counter() - t0
    atomic_write_text(report, report_text(preset, model.scenario(), threads, [
        ("command", "solve"), ("states", model.state_count()), ("actions", model.action_count()),
        ("outcomes", model.outcome_count()), ("iterations", res.iterations),
        ("converged", "true" if res.converged else "false"),
        ("precision", cfg.precision), ("resumed", "true" if resume else "false"),
        ("wall_seconds", format_double(wall))]))
    return SolveOutcome(model.state_count(), res.iterations, res.converged, wall, policy_csv,
                        ckpt, report)


def heuristic_params_text(model: P.Model, params) -> str:
    out = f"policy = {heuristic_kind(model)}\nfingerprint = {model.fingerprint().hex()}\n"
    for (name, _, _), v in zip(P.heuristic_space(model), params):
        out += f"{name} = {v}\n"
    return out


def heuristic_params_from_file(model: P.Model, path: str):
    try:
        text = open(path).read()
    except OSError as e:
        raise P.IoError(f"cannot open file: {path}") from e
    kv = {}
    for line in text.splitlines():
        if "=" in line:
            k, v = line.split("=", 1)
            kv[k.strip(" \t\r")] = v.strip(" \t\r")
    if "fingerprint" in kv and kv["fingerprint"] != model.fingerprint().hex():
        raise P.FingerprintMismatch(f"heuristic parameter fingerprint {kv['fingerprint']} does "
                                    f"not match the configured scenario's {model.fingerprint().hex()}")
    params = []
    for name, lo, hi in P.heuristic_space(model):
        if name not in kv:
            raise P.FormatError(f"heuristic parameter file is missing {name}")
        v = int(kv[name])
        if v < lo or v > hi:
            raise P.FormatError(f"heuristic parameter {name} out of range")
        params.append(v)
    return params


def cmd_simopt(preset: str, output_dir: str, threads: Optional[int] = None,
               rollouts_per_candidate: int = 4000, seed: int = 1, base_seed: int = 42,
               sampler: str = "auto"):
    """runner.cpp:352-439."""
    t0 = time.perf_counter()
    threads = threads or os.cpu_count() or 1
    os.makedirs(output_dir, exist_ok=True)
    model = P.make_preset(preset)
    space = P.heuristic_space(model)
    r = P.simopt(model, sampler=sampler, rollouts_per_candidate=rollouts_per_candidate,
                 seed=seed, base_seed=base_seed)
    used = sampler if sampler != "auto" else ("grid" if len(space) == 1 else "ga")
    log = csv_row(["generation"] + [n for n, _, _ in space] + ["mean_return", "sd_return"])
    for gen, vals, mean, sd in r.log:
        log += csv_row([gen] + list(vals) + [format_double(mean), format_double(sd)])
    atomic_write_text(os.path.join(output_dir, "search_log.csv"), log)
    atomic_write_text(os.path.join(output_dir, "best_params.txt"), heuristic_params_text(model, r.best))
    wall = time.perf_counter() - t0
    atomic_write_text(os.path.join(output_dir, "report.txt"), report_text(preset, model.scenario(), threads, [
        ("command", "simopt"), ("sampler", used), ("candidates_evaluated", len(r.log)),
        ("generations", r.generations if used == "ga" else 1),
        ("best_mean_return", format_double(r.best_mean)), ("wall_seconds", format_double(wall))]))
    return r


def kpi_header(products: int):
    h = ["policy", "return_mean", "return_sd"]
    suffixes = [""] if products == 1 else ["_a", "_b"]
    for sfx in suffixes:
        for base in ("service_pct", "wastage_pct", "holding"):
            h += [f"{base}{sfx}_mean", f"{base}{sfx}_sd"]
    return h + ["optimality_gap_pct"]


def kpi_row(name: str, ev: P.Evaluation, gap: Optional[float]):
    row = [name, format_double(ev.ret.mean), format_double(ev.ret.sd)]
    for k in range(ev.products):
        row += [format_double(ev.service_pct[k].mean), format_double(ev.service_pct[k].sd),
                format_double(ev.wastage_pct[k].mean), format_double(ev.wastage_pct[k].sd),
                format_double(ev.holding_mean[k].mean), format_double(ev.holding_mean[k].sd)]
    return row + [format_double(gap) if gap is not None else ""]


def cmd_evaluate(preset: str, output_dir: str, vi_policy: Optional[str] = None,
                 heuristic_params: Optional[str] = None, n_rollouts: int = 10_000,
                 base_seed: int = 42, horizon: int = 365, warmup: int = 100):
    """runner.cpp:441-480: both policies are scored in one device batch."""
    if not vi_policy and not heuristic_params:
        raise P.ConfigError("evaluate needs a policy CSV and/or a heuristic parameter file")
    os.makedirs(output_dir, exist_ok=True)
    model = P.make_preset(preset)
    cfg = P.RolloutConfig(horizon_days=horizon, warmup_days=warmup, n_rollouts=n_rollouts,
                          base_seed=base_seed)
    pols, names = [], []
    if vi_policy:
        pols.append(P.make_vi_policy(model, policy_from_csv(model, vi_policy)))
        names.append("value_iteration")
    if heuristic_params:
        pols.append(P.make_heuristic_policy(model, heuristic_params_from_file(model, heuristic_params)))
        names.append("heuristic")
    evs, _ = P.evaluate_policies(model, pols, cfg)
    out = dict(zip(names, evs))
    gap = None
    if len(evs) == 2:
        gap = 100.0 * (evs[0].ret.mean - evs[1].ret.mean) / abs(evs[0].ret.mean)
    csv = csv_row(kpi_header(model.products()))
    if "value_iteration" in out:
        csv += csv_row(kpi_row("value_iteration", out["value_iteration"], None))
    if "heuristic" in out:
        csv += csv_row(kpi_row("heuristic", out["heuristic"], gap))
    atomic_write_text(os.path.join(output_dir, "kpis.csv"), csv)
    return out, gap
