python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke21.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke21.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu21.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu21.log
timeout 600 python bench.py > gpurun_out/bench21.json 2>gpurun_out/bench21.err; echo bench=$?; cat gpurun_out/bench21.json; tail -3 gpurun_out/bench21.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench21_ref.json 2>gpurun_out/bench21_ref.err; echo ref=$?; cat gpurun_out/bench21_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches21.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c5 > /dev/null 2>&1; echo ncu=$?
