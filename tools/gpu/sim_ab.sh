for v in ${VALS:-1 2 3}; do echo "PVI_SIM_MINB=$v"; PVI_SIM_MINB=$v timeout 300 python tools/sim_ab.py; PVI_SIM_MINB=$v PVI_SIM_TRACE=1 python -c "
import sys; sys.path.insert(0,'.'); import paper_2303_10672_b200 as P
for pre, par in [('a/m5/exp5', lambda i:[i%11]), ('b/m2/exp1', lambda i:[i%21,(i*7)%21]), ('c/m3/exp1', lambda i:[(i+k)%10 for k in range(7)]+[(i+k)%10+10 for k in range(7)])]:
    m=P.make_preset(pre); pols=[P.make_heuristic_policy(m, par(i)) for i in range(50)]
    for _ in range(3): P.evaluate_policies(m, pols, P.RolloutConfig(n_rollouts=4096, base_seed=42))
" 2>&1 | grep "pvi sim" | awk 'NR%3==0'; done
