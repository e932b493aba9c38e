python -c "import paper_3004_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest30.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest30.log
timeout 300 python scripts/run_c5_distance.py 5 > gpurun_out/c5_30.json 2>&1; echo c5=$?; cat gpurun_out/c5_30.json | cut -c1-400
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof30_k_distance_c5 python scripts/run_c5_distance.py 1 > gpurun_out/prof30_c5.log 2>&1; echo ncu_c5=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches30_c5.csv python scripts/run_c5_distance.py 2 > /dev/null 2>&1; echo ncu_l=$?
