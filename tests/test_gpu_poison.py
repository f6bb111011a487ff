"""compute-sanitizer stand-in (the tool is closed on this
GPU pool: gpurun_out logs "compute-sanitizer is closed on this pool").

Each case runs in a subprocess with PVI_POISON=1, which fills every sweep
scratch buffer (W, G, the binomial-pass tables, partial maxima) and every
output slice with 0xFF bytes (NaN / action 255) before each sweep.  A kernel
that reads an element no kernel wrote this sweep, or leaves an output element
unwritten, then produces NaN or a wrong action: the results must equal the
unpoisoned run bit for bit.  Covers the factored kernels the verdict names
(k_b_fact_w16p, k_b_fact_qw4, k_c_fact_g, k_c_bin_tile_p, k_c_bin_qf /
k_c_bin_q, k_a_fact_*) plus the exact kernels and Q-row queries."""
import hashlib
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2303_10672_b200 as P
preset, algo, lo, hi, q = sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]), sys.argv[6] == "q"
m = P.make_preset(preset).set_algorithm(algo)
n = m.state_count()
hi = n if hi < 0 else hi
V = np.random.default_rng(4).uniform(-10.0, 10.0, n)
h = hashlib.sha256()
for _ in range(2):
    if q:
        h.update(P.q_rows(m, V, lo, hi).tobytes())
    else:
        v, a = P.bellman_backup_batch(m, V, lo, hi)
        assert np.isfinite(v).all(), "non-finite output"
        h.update(v.tobytes()); h.update(a.tobytes())
print(h.hexdigest())
'''

CASES = [("b/m3/exp1", "factored", 0, -1, ""), ("b/m3/exp1", "factored", 3 << 20, 5 << 20, ""),
         ("b/m2/exp1", "factored", 0, -1, ""), ("b/m3/exp4", "factored", 0, -1, ""),
         ("b/m3/exp1", "factored", 1000, 1200, "q"), ("c/m5/exp1", "factored", 0, -1, ""),
         ("c/m5/exp2", "factored", 0, -1, ""), ("c/m3/exp2", "factored", 0, -1, ""),
         ("c/m5/exp2", "factored", 500000, 500300, "q"), ("a/m5/exp5", "factored", 0, -1, ""),
         ("a/m5/exp6", "factored", 0, -1, ""), ("b/m2/exp1", "exact", 0, -1, ""),
         ("c/m3/exp1", "exact", 0, -1, ""), ("a/m3/exp5", "exact", 0, -1, "")]


def _run(case, poison):
    env = dict(os.environ, PVI_POISON="1" if poison else "0")
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT] + [str(x) for x in case],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout.strip().splitlines()[-1]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "-".join(str(x) for x in c if x != ""))
def test_poisoned_scratch_changes_nothing(case):
    assert _run(case, True) == _run(case, False)
