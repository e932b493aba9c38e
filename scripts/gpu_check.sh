python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_check.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_check.log; grep -m2 -A25 "FAILED\|Error" gpurun_out/pytest_check.log | head -40
