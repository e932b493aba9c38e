python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest42.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest42.log
timeout 300 python scripts/run_c5_generation.py 3 > gpurun_out/c5g42.json 2>&1; echo c5g=$?; tail -c 600 gpurun_out/c5g42.json
