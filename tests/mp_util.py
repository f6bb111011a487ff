"""Collect results of spawned rank processes without hanging on a dead one."""
import queue
import time


def collect(procs, q, n, timeout):
    """n results from q; fails as soon as a rank process exits non-zero
    (instead of waiting out the whole timeout), or after `timeout` s."""
    out = []
    deadline = time.time() + timeout
    while len(out) < n:
        try:
            out.append(q.get(timeout=2.0))
            continue
        except queue.Empty:
            pass
        dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
        if dead:
            for p in procs:
                if p.is_alive():
                    p.terminate()
            raise AssertionError(f"a rank process failed (exit codes {[p.exitcode for p in procs]})")
        if time.time() > deadline:
            for p in procs:
                if p.is_alive():
                    p.terminate()
            raise AssertionError(f"timed out after {timeout} s waiting for {n - len(out)} rank results")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, [p.exitcode for p in procs]
    return out
