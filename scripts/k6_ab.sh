# K6 attrs A/B at C5: kernel durations (ncu launch list, cold-cache) of the
# HEAD build in ab_old/ (git worktree) against the working tree, then parity
export FNB_STEP_GRAPH=0 FNB_GEN_GRAPH=0
for side in ${SIDES:-old new}; do
  # old: the HEAD build in ab_old/; newB: ab_b/; off: the working tree with the prefetch knobs off
  unset FNB_AB_ROOT FNB_XOVER_L2PF FNB_K6_L2PF FNB_K1_L2PF
  case $side in
    old) export FNB_AB_ROOT=$GRAFT_REPO_ROOT/ab_old ;;
    newB) export FNB_AB_ROOT=$GRAFT_REPO_ROOT/ab_b ;;
    ab_*) export FNB_AB_ROOT=$GRAFT_REPO_ROOT/$side ;;
    off) export FNB_XOVER_L2PF=0 FNB_K6_L2PF=0 ;;
  esac
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg --clock-control none -k regex:"k_mutate|k_crossover|k_transform" --csv \
    --log-file gpurun_out/k6ab_$side.csv python scripts/run_c5_generation.py 2 > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg --clock-control none -k regex:"k_mutate|k_crossover|k_transform|k_distance" --csv \
    --log-file gpurun_out/k6ab_${side}_c2.csv python scripts/run_c2_generation.py 4 > /dev/null 2>&1
  for f in $side ${side}_c2; do python - $f <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/k6ab_{sys.argv[1]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); mi = h.index("Metric Name")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[(r[ki].split("(")[0], r[mi])].append(float(r[vi].replace(",", "")))
print(sys.argv[1], {k[0] + (" ms" if "time" in k[1] else " Mcyc"): round(sum(v) / len(v) / 1e6, 4) for k, v in d.items() if "time" in k[1]})
PY
  done
done
unset FNB_STEP_GRAPH FNB_GEN_GRAPH FNB_AB_ROOT FNB_XOVER_L2PF FNB_K6_L2PF
timeout 900 python -m pytest tests/test_gpu_mutate.py tests/test_gpu_evolve.py tests/test_gpu_c5_scale.py -q -x 2>&1 | tail -2
