"""SHA-256 of one full factored sweep (V', argmax) of the C presets, to
compare the binomial-pass kernels bit for bit across PVI_C_TILE modes:
  for t in 2 3; do PVI_C_TILE=$t python tools/c_tile_hash.py; done"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_10672_b200 as P  # noqa: E402

for preset in ("c/m3/exp1", "c/m3/exp2", "c/m5/exp1", "c/m5/exp2"):
    m = P.make_preset(preset).set_algorithm("factored")
    r = P.run_value_iteration(m, P.ViConfig(fixed_iterations=3))
    h = hashlib.sha256(r.values.tobytes() + r.policy.tobytes()).hexdigest()[:16]
    print(os.environ.get("PVI_C_TILE", "default"), preset, h, flush=True)
