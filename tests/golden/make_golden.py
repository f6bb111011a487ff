"""Generate tests/golden/*.npz from the UNMODIFIED reference.

Run in the build container (it needs oracle/_ref/libpvi_ref.so, which is
compiled from /root/reference by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every array here is an output of the reference library itself (through
oracle/ref_capi.cpp), never of the code under test.  The GPU box has no
/root/reference, so these fixtures are what the parity tests travel with.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

SOLVES = [("a/m2/exp1", False), ("a/m2/exp2", False), ("a/m2/exp6", False),
          ("a/m3/exp5", False), ("b/m2/exp1", False), ("b/m2/exp2", False),
          ("c/m3/exp1", False), ("c/m3/exp2", False), ("a/m2/exp1", True),
          ("c/m3/exp1", True)]
FIXED = [("b/m2/p1", 100), ("b/m2/p4", 100), ("b/m3/exp4", 2)]
QROWS = {"b/m3/exp1": [0, 1, 4095, 65536 * 7 + 1234, 8388608 + 777, 16777215],
         "b/m3/exp4": [0, 5000, 777777, 1157624],
         "c/m5/exp1": [0, 1, 700000, 1361366],
         "c/m5/exp2": [123456],
         "a/m5/exp5": [0, 999999, 1771560],
         "a/m5/exp8": [31337]}
HEURISTICS = [("a/m2/exp1", [5]), ("a/m3/exp6", [7]), ("a/m5/exp5", [9]),
              ("b/m2/exp1", [13, 12]), ("b/m3/exp4", [25, 7]),
              ("c/m3/exp1", [9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8]),
              ("c/m5/exp2", [3, 4, 5, 6, 7, 2, 1, 10, 11, 12, 13, 14, 8, 9])]
TABULAR = [(30, 4, 5, 0.9, 1234), (20, 3, 4, 0.9, 555), (15, 3, 4, 0.9, 808),
           (12, 3, 4, 0.85, 2712), (64, 2, 2, 0.9, 3)]


def main():
    assert R.available(), "build oracle/_ref first: make -C oracle ref"
    out = {}
    for preset, f32 in SOLVES:
        s = R.vi_solve(preset, f32=f32)
        key = f"solve|{preset}|{'f32' if f32 else 'f64'}"
        out[key + "|values"] = s.values
        out[key + "|policy"] = s.policy
        out[key + "|meta"] = np.array([s.iterations, int(s.converged)], np.int64)
    for preset, k in FIXED:
        s = R.vi_solve(preset, fixed_iterations=k)
        key = f"fixed|{preset}|{k}"
        if len(s.values) > 100_000:  # large: SHA-256 of the raw bytes + a sample
            out[key + "|values_sha256"] = np.frombuffer(hashlib.sha256(s.values.tobytes()).digest(), np.uint8)
            out[key + "|policy_sha256"] = np.frombuffer(hashlib.sha256(s.policy.tobytes()).digest(), np.uint8)
            pick = np.arange(0, len(s.values), 997)
            out[key + "|sample_states"] = pick
            out[key + "|sample_values"] = s.values[pick]
        else:
            out[key + "|values"] = s.values
            out[key + "|policy"] = s.policy
    for preset, states in QROWS.items():
        n = R.counts(preset).states
        V = np.random.default_rng(7).uniform(-5.0, 5.0, n)
        qs = np.stack([R.q_row(preset, s, V) for s in states])
        out[f"qrow|{preset}|states"] = np.array(states, np.int64)
        out[f"qrow|{preset}|q"] = qs
        out[f"qrow|{preset}|naive"] = np.stack([R.naive_q_row(preset, s, V) for s in states[:2]])
    out["v0|b/m2/exp1"] = R.initial_values("b/m2/exp1")
    v0 = R.initial_values("b/m3/exp4")
    pick = np.arange(0, len(v0), 997)
    out["v0sample|b/m3/exp4|states"] = pick
    out["v0sample|b/m3/exp4|values"] = v0[pick]
    for preset, params in HEURISTICS:
        pr, ev = R.eval_heuristic(preset, params, 512, seed=42)
        out[f"sim|{preset}|{','.join(map(str, params))}|rollouts"] = pr
        out[f"sim|{preset}|{','.join(map(str, params))}|eval"] = ev
    s = R.vi_solve("a/m2/exp1")
    pr, ev = R.eval_table("a/m2/exp1", s.policy, 2000, seed=42)
    out["simvi|a/m2/exp1|rollouts"] = pr
    out["simvi|a/m2/exp1|eval"] = ev
    s = R.vi_solve("b/m2/exp1")
    pr, ev = R.eval_table("b/m2/exp1", s.policy, 1000, seed=42)
    out["simvi|b/m2/exp1|rollouts"] = pr
    out["simvi|b/m2/exp1|policy"] = s.policy
    for ns, na, no, g, seed in TABULAR:
        nxt, rew, prob = R.tabular_random(ns, na, no, g, seed)
        key = f"tab|{ns}|{na}|{no}|{g}|{seed}"
        out[key + "|next"], out[key + "|reward"], out[key + "|prob"] = nxt, rew, prob
        s = R.tabular_solve(ns, na, no, g, nxt, rew, prob, epsilon=1e-12)
        out[key + "|values"], out[key + "|policy"] = s.values, s.policy
        out[key + "|meta"] = np.array([s.iterations, int(s.converged)], np.int64)
        if ns <= 8:
            bv, bp = R.tabular_brute_force(ns, na, no, g, nxt, rew, prob)
            out[key + "|brute_values"], out[key + "|brute_policy"] = bv, bp
    # brute-force policy trials (test_vi.cpp:74-91 style, seeds drawn here)
    rng = np.random.default_rng(2024)
    for t in range(10):
        ns, na, seed = int(3 + rng.integers(6)), int(2 + rng.integers(2)), int(rng.integers(1 << 31))
        nxt, rew, prob = R.tabular_random(ns, na, 4, 0.9, seed)
        key = f"brute|{t}"
        out[key + "|dims"] = np.array([ns, na, 4, seed], np.int64)
        out[key + "|next"], out[key + "|reward"], out[key + "|prob"] = nxt, rew, prob
        s = R.tabular_solve(ns, na, 4, 0.9, nxt, rew, prob, epsilon=1e-12)
        bv, bp = R.tabular_brute_force(ns, na, 4, 0.9, nxt, rew, prob)
        out[key + "|values"], out[key + "|policy"] = s.values, s.policy
        out[key + "|brute_values"], out[key + "|brute_policy"] = bv, bp
    # tables
    out["table|a/m2/exp1|a.pmf"] = R.table_a_pmf("a/m2/exp1")
    for preset in ["b/m2/exp1", "b/m3/exp1", "b/m3/exp4"]:
        t = R.b_tables(preset)
        for k in ["pu", "pz", "pz_cum"]:
            out[f"table|{preset}|b.{k}"] = t[k].ravel()
        out[f"table|{preset}|caps"] = np.array([t["max_order_a"], t["max_order_b"]], np.int64)
        out[f"issued|{preset}|4095"] = R.b_issued_pmf(preset, 4095 % R.counts(preset).states)
    for preset in ["c/m3/exp1", "c/m3/exp2", "c/m5/exp1", "c/m5/exp2"]:
        t = R.c_tables(preset)
        out[f"table|{preset}|c.pmf"] = t["weekday_pmf"].ravel()
        out[f"table|{preset}|c.comp_probs"] = t["probs"]
    # RNG known answers
    out["philox|zero"] = R.philox_block([0] * 4, [0] * 2)
    out["philox|ones"] = R.philox_block([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)
    out["philox|pi"] = R.philox_block([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                                      [0xa4093822, 0x299f31d0])
    out["draws|42|0|0"] = R.rollout_draws(42, 0, 0, 8)
    out["draws|99|17|364"] = R.rollout_draws(99, 17, 364, 8)
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


def simopt_golden():
    """cmd_simopt trajectories (runner.cpp:352-403) with 4096 rollouts per
    candidate, eval seed 42, GA seed 1."""
    out = {}
    for preset in ["a/m2/exp1", "b/m2/exp1", "c/m3/exp1"]:
        r = R.simopt(preset, rollouts=4096, eval_seed=42, ga_seed=1)
        dim = {"a": 1, "b": 2, "c": 14}[preset[0]]
        n = r["n_logged"]
        out[f"simopt|{preset}|best"] = r["best"][:dim].astype(np.int64)
        out[f"simopt|{preset}|meta"] = np.array([r["generations"], n], np.int64)
        out[f"simopt|{preset}|score"] = np.array([r["mean"], r["sd"]])
        out[f"simopt|{preset}|log_values"] = r["log_values"][:n * dim].reshape(n, dim).astype(np.int64)
        out[f"simopt|{preset}|log_scores"] = r["log_scores"][:n]
        out[f"simopt|{preset}|ref_wall"] = np.array([r["wall"]])
        print(preset, r["best"][:dim], r["mean"], r["generations"], n, r["wall"])
    np.savez_compressed(os.path.join(HERE, "simopt_golden.npz"), **out)


RUNNER_CASES = [("a/m2/exp1", 4096, 2000), ("b/m2/exp1", 4096, 1000), ("c/m3/exp1", 0, 500)]


def runner_golden():
    """Files written by the reference runner's cmd_solve / cmd_simopt /
    cmd_evaluate (runner.cpp:303-480) for small presets."""
    import ctypes as C
    import tempfile
    L = R.lib()
    L.ref_cmd.argtypes = [C.c_char_p, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_char_p,
                          C.c_char_p, C.c_char_p, C.c_size_t]
    out = {}
    err = C.create_string_buffer(1024)
    for preset, simopt_rollouts, eval_rollouts in RUNNER_CASES:
        d = tempfile.mkdtemp()
        assert L.ref_cmd(preset.encode(), 0, d.encode(), 8, 0, b"", b"", err, 1024) == 0, err.value
        heur = b""
        if simopt_rollouts:
            assert L.ref_cmd(preset.encode(), 1, d.encode(), 8, simopt_rollouts, b"", b"", err,
                             1024) == 0, err.value
            heur = (d + "/best_params.txt").encode()
        else:  # c/m3: the published weekday (s, S) table (PAPER Table 13 exp1)
            vals = [9, 7, 7, 6, 6, 3, 3, 13, 14, 14, 10, 11, 8, 8]
            names = [f"s.{t}" for t in range(7)] + [f"S.{t}" for t in range(7)]
            with open(d + "/heuristic.txt", "w") as f:
                f.write("policy = weekday_sS\n" + "".join(f"{n} = {v}\n" for n, v in zip(names, vals)))
            heur = (d + "/heuristic.txt").encode()
        assert L.ref_cmd(preset.encode(), 2, d.encode(), 8, eval_rollouts,
                         (d + "/policy.csv").encode(), heur, err, 1024) == 0, err.value
        for fn in sorted(os.listdir(d)):
            if fn.endswith(".tmp"):
                continue
            data = open(os.path.join(d, fn), "rb").read()
            if fn == "report.txt":  # drop the machine-dependent lines
                data = b"".join(l for l in data.splitlines(True)
                                if not l.startswith((b"wall_seconds", b"threads")))
            out[f"runner|{preset}|{fn}"] = np.frombuffer(data, np.uint8)
        print(preset, sorted(os.listdir(d)))
    np.savez_compressed(os.path.join(HERE, "runner_golden.npz"), **out)


def runner_large_golden():
    """acceptance_main.cpp:303-325: b/m3/exp4 (1.16M states) cmd_solve with
    3 fixed sweeps, uninterrupted and as 2 + resume; SHA-256 of the files
    (the policy CSV is ~30 MB)."""
    import ctypes as C
    import hashlib
    import tempfile
    L = R.lib()
    L.ref_cmd_solve_fixed.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64, C.c_int, C.c_char_p,
                                      C.c_size_t]
    err = C.create_string_buffer(1024)
    out = {}
    d_ref, d_res = tempfile.mkdtemp(), tempfile.mkdtemp()
    assert L.ref_cmd_solve_fixed(b"b/m3/exp4", d_ref.encode(), 8, 3, 0, err, 1024) == 0, err.value
    assert L.ref_cmd_solve_fixed(b"b/m3/exp4", d_res.encode(), 8, 2, 0, err, 1024) == 0, err.value
    assert L.ref_cmd_solve_fixed(b"b/m3/exp4", d_res.encode(), 8, 3, 1, err, 1024) == 0, err.value
    for fn in ["checkpoint.ckpt", "policy.csv"]:
        a = open(os.path.join(d_ref, fn), "rb").read()
        b = open(os.path.join(d_res, fn), "rb").read()
        assert a == b, fn  # the reference's own clause
        out[f"runner_large|b/m3/exp4|3|{fn}|sha256"] = np.frombuffer(hashlib.sha256(a).digest(), np.uint8)
        out[f"runner_large|b/m3/exp4|3|{fn}|bytes"] = np.array([len(a)], np.int64)
    np.savez_compressed(os.path.join(HERE, "runner_large_golden.npz"), **out)
    print("runner_large", {k: v.tolist() for k, v in out.items() if k.endswith("bytes")})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "simopt":
        simopt_golden()
    elif len(sys.argv) > 1 and sys.argv[1] == "runner":
        runner_golden()
    elif len(sys.argv) > 1 and sys.argv[1] == "runner_large":
        runner_large_golden()
    else:
        main()
