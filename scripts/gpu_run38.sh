python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches38_c5g.csv python scripts/run_c5_generation.py 2 > gpurun_out/c5g38.log 2>&1; echo ncu=$?; tail -2 gpurun_out/c5g38.log
