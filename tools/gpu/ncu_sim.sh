# ncu of the rollout kernel behind simopt (config 5: b/m2/exp1 GA, 4096 rollouts/candidate)
mkdir -p gpurun_out
S="python -c \"import sys; sys.path.insert(0,'.'); import paper_2303_10672_b200 as P; r=P.simopt(P.make_preset('b/m2/exp1'), rollouts_per_candidate=4096, base_seed=42, seed=1); print(len(r.log), r.device_seconds)\""
eval $S > gpurun_out/sim_plain.log 2>&1 && \
  eval ncu --set full --clock-control none --import-source on -k regex:k_rollouts -s 1 -c 1 -o gpurun_out/k5 $S > gpurun_out/ncu_k5.log 2>&1
python tools/ncu_summary.py gpurun_out/k5.ncu-rep gpurun_out/r1b_k5_simopt_ncu.json
ncu -i gpurun_out/k5.ncu-rep --page details --csv > gpurun_out/k5_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/sim_plain.log
