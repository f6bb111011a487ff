PVI_LOOP_TRACE=1 python - <<'P'
import sys, time
sys.path.insert(0, ".")
import paper_2303_10672_b200 as P
for preset, algo in [("a/m5/exp5", "factored"), ("b/m3/exp1", "factored")]:
    m = P.make_preset(preset).set_algorithm(algo)
    P.run_value_iteration(m, P.ViConfig(fixed_iterations=2))
    for loop in ("host", "graph", "host", "graph"):
        t = time.perf_counter()
        r = P.run_value_iteration(m, P.ViConfig(loop=loop, l2_persist=False))
        print(preset, loop, r.iterations, f"wall {r.wall_seconds*1e3:.1f} ms py {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
P
