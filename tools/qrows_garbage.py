"""Q rows (exact and factored) after the device memory was filled with
garbage: a read of uninitialised scratch shows up as a mismatch against the
C oracle.  Usage: python tools/qrows_garbage.py [preset ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2303_10672_b200 as pvi  # noqa: E402
from oracle import cport  # noqa: E402


def poison(gib=60, pattern=float("nan")):
    x = torch.full((gib << 27,), pattern, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()


def main():
    presets = sys.argv[1:] or ["c/m5/exp1", "c/m5/exp2"]
    for pattern in (float("nan"), 1e300, 0.0):
        poison(pattern=pattern)
        for preset in presets:
            for prec in ("f64", "f32"):
                exact = pvi.make_preset(preset)
                fact = pvi.make_preset(preset).set_algorithm("factored")
                n = exact.state_count()
                V = np.random.default_rng(9).uniform(-50.0, 50.0, n)
                lo = n // 2
                hi = min(n, lo + 512)
                qe = pvi.q_rows(exact, V, lo, hi, precision=prec).astype(np.float64)
                qf = pvi.q_rows(fact, V, lo, hi, precision=prec).astype(np.float64)
                tol = 1e-12 if prec == "f64" else 2e-6
                bad = ~np.isclose(qf, qe, rtol=tol, atol=tol * 100)
                msg = f"{pattern} {preset} {prec}: {int(bad.sum())} mismatches"
                for s_off, a in zip(*np.nonzero(bad)):
                    s = lo + int(s_off)
                    ref = cport.q_row(preset, s, V,
                                      f32=prec == "f32")
                    msg += (f"\n   s={s} a={a} exact={qe[s_off, a]!r} factored={qf[s_off, a]!r}"
                            f" oracle={float(ref[a])!r}")
                print(msg, flush=True)


if __name__ == "__main__":
    main()
