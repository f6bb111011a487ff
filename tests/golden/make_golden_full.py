"""Full-size one-sweep fixtures for the headline presets, from the UNMODIFIED
reference (oracle/_ref, `bellman_backup_batch` over every state,
vi.hpp:82-92 driven as run_value_iteration's sweep body vi.hpp:231-243).

    python tests/golden/make_golden_full.py [preset ...]

Each case is one Jacobi sweep over the whole state space from a fixed input
vector: V0 = ScenarioB::initial_value for b/m3/exp1 (the solve's first sweep,
SURVEY App. B), and a seeded uniform(-5, 5) vector (numpy default_rng(7),
reproducible on the GPU box) for the others.  Stored per case: SHA-256 of
the f64 values and of the u32 argmax vector, and every 997th state's value
and action — enough to pin a GPU sweep bit for bit without shipping 200 MB.
Takes ~15 min (b/m3/exp1) and ~45 min per c/m5 preset on 8 cores.
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import refbind as R  # noqa: E402

CASES = {"b/m3/exp1": "v0", "a/m5/exp5": "rand7", "a/m5/exp6": "rand7",
         "c/m5/exp1": "rand7", "c/m5/exp2": "rand7"}
OUT = os.path.join(HERE, "full_sweeps.npz")


def input_vector(preset: str, kind: str, n: int) -> np.ndarray:
    if kind == "v0":
        return R.initial_values(preset)
    return np.random.default_rng(7).uniform(-5.0, 5.0, n)


def main(presets):
    out = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    for preset in presets:
        kind = CASES[preset]
        n = R.counts(preset).states
        V = input_vector(preset, kind, n)
        t0 = time.time()
        vals, acts, secs = R.backup_range(preset, V, 0, n)
        key = f"full|{preset}|{kind}"
        out[key + "|values_sha256"] = np.frombuffer(hashlib.sha256(vals.tobytes()).digest(), np.uint8)
        out[key + "|actions_sha256"] = np.frombuffer(hashlib.sha256(acts.tobytes()).digest(), np.uint8)
        pick = np.arange(0, n, 997)
        out[key + "|sample_states"] = pick
        out[key + "|sample_values"] = vals[pick]
        out[key + "|sample_actions"] = acts[pick]
        out[key + "|ref_seconds"] = np.array([secs, float(R.hardware_threads())])
        np.savez_compressed(OUT, **out)
        print(f"{preset} {kind}: {n} states, {secs:.1f} s ({time.time() - t0:.1f} s wall), "
              f"V[0]={vals[0]!r} V[-1]={vals[-1]!r}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
