# round-1 profile set: full bench line, launch list, ncu --set full of the K2 / K3(C5) / C4 rollout / K6 kernels
python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python bench.py > gpurun_out/bench36.json 2>gpurun_out/bench36.err; echo bench=$?; tail -2 gpurun_out/bench36.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches36.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_forward --launch-skip 4 -c 1 -f -o gpurun_out/prof36_k2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof36_k3_c5 python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hyper_rollout -c 1 -f -o gpurun_out/prof36_c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-generations > /dev/null 2>&1; echo ncu_c4=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mutate_attrs --launch-skip 3 -c 1 -f -o gpurun_out/prof36_k6 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 > /dev/null 2>&1; echo ncu_k6=$?
