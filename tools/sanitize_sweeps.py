"""One factored sweep of a small case, for compute-sanitizer (VERDICT r1
item 2).  Usage: python tools/sanitize_sweeps.py CASE
CASE: b_m2 | c_m3_exp1 | c_m3_exp2 | b_m3_slice | c_m5_exp2_q | a_m4_fifo
Each runs the factored sweep twice on the same V and checks the two results
are identical (a race would usually show up as a difference as well)."""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2303_10672_b200 as P  # noqa: E402

CASES = {
    "b_m2": ("b/m2/exp1", None),            # k_b_fact_w + k_b_fact_q (generic radix)
    "c_m3_exp1": ("c/m3/exp1", None),       # k_c_fact_g + k_c_bin_tile_p<21> + k_c_bin_qf<21>
    "c_m3_exp2": ("c/m3/exp2", None),       # endogenous: k_c_bin_tile_p + k_c_bin_q + k_finalize
    "b_m3_slice": ("b/m3/exp1", (0, 1 << 17)),  # k_b_fact_w16p + k_b_fact_qw4, one x_3 pair
    "a_m4_fifo": ("a/m4/exp2", None),       # k_a_fact_fifo
    "a_m4_lifo": ("a/m4/exp1", None),       # k_a_fact_lifo
}


def main(case):
    preset, rng = CASES[case]
    m = P.make_preset(preset).set_algorithm("factored")
    n = m.state_count()
    lo, hi = rng or (0, n)
    V = np.random.default_rng(1).uniform(-10.0, 10.0, n)
    h = set()
    for _ in range(2):
        v, a = P.bellman_backup_batch(m, V, lo, hi)
        h.add(hashlib.sha256(v.tobytes() + a.tobytes()).hexdigest())
    assert len(h) == 1, f"{case}: repeated sweeps differ"
    print(f"{case}: {preset} [{lo}, {hi}) ok {next(iter(h))[:16]}")


if __name__ == "__main__":
    main(sys.argv[1])
