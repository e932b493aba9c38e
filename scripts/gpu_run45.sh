python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest45.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest45.log
timeout 300 python scripts/run_c5_generation.py 3 > gpurun_out/c5g45.json 2>&1; echo c5g=$?; tail -c 500 gpurun_out/c5g45.json
timeout 600 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/bench45.json 2>gpurun_out/bench45.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench45.json'));print(d['generations'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches45_c5g.csv python scripts/run_c5_generation.py 1 > /dev/null 2>&1; echo ncu=$?
