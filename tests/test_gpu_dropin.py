"""The reference-side drop-in (include/pvi/b200.hpp), compiled against the
unmodified reference (make -C oracle dropin, in the build container) and run
here on the GPU: every case compares the reference's own template with the
pvi::b200 overload bit for bit (tests/dropin/dropin_main.cpp)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_test")


def test_dropin_against_reference():
    assert os.path.exists(BIN), "oracle/_ref/dropin_test missing: build() compiles it (make -C oracle dropin)"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1200)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
    assert "dropin: " in r.stdout and " 0 failed" in r.stdout
