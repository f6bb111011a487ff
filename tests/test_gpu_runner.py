"""cmd_solve / cmd_simopt / cmd_evaluate (runner.cpp:303-480) over the B200
engine write the reference runner's files byte for byte:
checkpoint.ckpt, policy.csv (+ .meta.json), search_log.csv, best_params.txt,
kpis.csv and report.txt (minus its wall-clock and thread-count lines).
Expected files: tests/golden/runner_golden.npz (the reference runner's
output, tests/golden/make_golden.py runner)."""
import os
import shutil

import numpy as np
import pytest

from paper_2303_10672_b200 import runner

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "runner_golden.npz"))
CASES = [("a/m2/exp1", 4096, 2000), ("b/m2/exp1", 4096, 1000), ("c/m3/exp1", 0, 500)]


def _strip(data: bytes) -> bytes:
    return b"".join(l for l in data.splitlines(True) if not l.startswith((b"wall_seconds", b"threads")))


@pytest.mark.parametrize("preset,simopt_rollouts,eval_rollouts", CASES)
def test_runner_files_match_reference(tmp_path, preset, simopt_rollouts, eval_rollouts):
    d = str(tmp_path)
    runner.cmd_solve(preset, d)
    if simopt_rollouts:
        runner.cmd_simopt(preset, d, rollouts_per_candidate=simopt_rollouts)
        heur = os.path.join(d, "best_params.txt")
    else:
        heur = os.path.join(d, "heuristic.txt")
        open(heur, "wb").write(bytes(G[f"runner|{preset}|heuristic.txt"]))
    runner.cmd_evaluate(preset, d, vi_policy=os.path.join(d, "policy.csv"),
                        heuristic_params=heur, n_rollouts=eval_rollouts)
    names = sorted(k.split("|")[2] for k in G.files if k.startswith(f"runner|{preset}|"))
    assert sorted(f for f in os.listdir(d) if not f.endswith(".tmp")) == names
    for fn in names:
        got = open(os.path.join(d, fn), "rb").read()
        want = bytes(G[f"runner|{preset}|{fn}"])
        if fn == "report.txt":
            got = _strip(got)
        assert got == want, fn


def test_resume_from_runner_checkpoint(tmp_path):
    d = str(tmp_path)
    runner.cmd_solve("a/m2/exp1", d)
    first = open(os.path.join(d, "policy.csv"), "rb").read()
    runner.cmd_solve("a/m2/exp1", d, resume=True)  # converged checkpoint: one more check
    assert "resumed = true" in open(os.path.join(d, "report.txt")).read()
    assert open(os.path.join(d, "policy.csv"), "rb").read() == first


def test_evaluate_refuses_foreign_policy(tmp_path, pvi):
    d = str(tmp_path)
    runner.cmd_solve("a/m2/exp1", d)
    shutil.copy(os.path.join(d, "policy.csv.meta.json"), os.path.join(d, "x.meta.json"))
    with pytest.raises(pvi.FingerprintMismatch):
        runner.cmd_evaluate("a/m2/exp2", d, vi_policy=os.path.join(d, "policy.csv"), n_rollouts=10)


LARGE = np.load(os.path.join(os.path.dirname(__file__), "golden", "runner_large_golden.npz"))


@pytest.mark.parametrize("algorithm", ["exact", "factored"])
def test_b_m3_exp4_command_level_resume_bitwise(tmp_path, algorithm):
    """acceptance_main.cpp:303-325: b/m3/exp4 (1.16M states), cmd_solve with
    3 fixed sweeps, uninterrupted vs 2 sweeps + resume: the checkpoint and
    policy CSV files are identical.  On the exact path both also equal the
    reference runner's files byte for byte (SHA-256 fixture)."""
    import hashlib
    from paper_2303_10672_b200 import runner
    import paper_2303_10672_b200 as P
    ref_dir, res_dir = str(tmp_path / "ref"), str(tmp_path / "res")
    runner.cmd_solve("b/m3/exp4", ref_dir, threads=8, config=P.ViConfig(fixed_iterations=3), algorithm=algorithm)
    runner.cmd_solve("b/m3/exp4", res_dir, threads=8, config=P.ViConfig(fixed_iterations=2), algorithm=algorithm)
    runner.cmd_solve("b/m3/exp4", res_dir, threads=8, config=P.ViConfig(fixed_iterations=3), resume=True,
                     algorithm=algorithm)
    for fn in ["checkpoint.ckpt", "policy.csv"]:
        a = open(os.path.join(ref_dir, fn), "rb").read()
        b = open(os.path.join(res_dir, fn), "rb").read()
        assert a == b, fn
        if algorithm == "exact":
            assert len(a) == int(LARGE[f"runner_large|b/m3/exp4|3|{fn}|bytes"][0])
            assert hashlib.sha256(a).digest() == LARGE[f"runner_large|b/m3/exp4|3|{fn}|sha256"].tobytes(), fn
