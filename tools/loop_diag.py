import sys, os
sys.path.insert(0, os.getcwd())
import paper_2303_10672_b200 as P
for preset, algo, test in [("c/m3/exp1", "exact", "change_span"), ("c/m3/exp1", "factored", "change_span"),
                           ("c/m3/exp1", "exact", None), ("a/m2/exp1", "exact", "periodic_span")]:
    m = P.make_preset(preset).set_algorithm(algo)
    try:
        r = P.run_value_iteration(m, P.ViConfig(loop="graph", convergence_test=test))
        print(preset, algo, test, "ok", r.iterations, r.graph_sweeps, flush=True)
    except Exception as e:
        print(preset, algo, test, "FAIL", e, flush=True)
