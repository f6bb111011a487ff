import sys, time
sys.path.insert(0, '.')
import paper_2303_10672_b200 as P
for preset in ["a/m2/exp1", "a/m2/exp2", "a/m2/exp1", "a/m2/exp2", "a/m3/exp5"]:
    for algo in ["exact", "factored"]:
        m = P.make_preset(preset).set_algorithm(algo)
        t = time.perf_counter()
        r = P.run_value_iteration(m)
        w = time.perf_counter() - t
        print(preset, algo, r.iterations, f"wall {r.wall_seconds:.4f} call {w:.4f} sweep_s {r.sweep_seconds:.4f} graph_sweeps {r.graph_sweeps}", flush=True)
