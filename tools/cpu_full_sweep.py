"""Validate the bench's tile-sampled CPU baseline against one FULL reference
sweep.  Runs on the GPU box's host
cores (nothing here touches the GPU):

    python tools/cpu_full_sweep.py [preset] > gpurun_out/cpu_full_sweep.json

1. the bench's sampled estimate (bench.run_cpu_reference, 12 s budget);
2. the reference's bellman_backup_batch over ALL states from V0, all cores;
prints both rates and their ratio as one JSON object."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from oracle import refbind as R  # noqa: E402


def main(preset="b/m3/exp1"):
    work = bench.work_from_reference(preset)
    V = R.initial_values(preset)
    rate_s, secs_s, terms_s, desc, threads = bench.run_cpu_reference(work, preset, "f64", 12.0, V)
    t0 = time.time()
    vals, acts, secs = R.backup_range(preset, V, 0, work.states, threads=threads)
    wall = time.time() - t0
    rate_f = work.terms / secs
    print(json.dumps({"preset": preset, "threads": threads, "terms_per_sweep": work.terms,
                      "sampled": {"evals_per_s": rate_s, "seconds": secs_s, "terms": terms_s,
                                  "sample": desc},
                      "full_sweep": {"evals_per_s": rate_f, "seconds": secs, "wall_seconds": wall,
                                     "V1_0": float(vals[0]), "V1_last": float(vals[-1])},
                      "sampled_over_full": rate_s / rate_f,
                      "host": os.uname().nodename, "cpu_count": os.cpu_count()}))


if __name__ == "__main__":
    main(*sys.argv[1:])
