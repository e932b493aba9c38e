python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest52.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest52.log
timeout 600 python bench.py --no-cpu-baseline --no-c5 > gpurun_out/bench52.json 2>gpurun_out/bench52.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench52.json'));print(d['generations']['ms_per_generation'], d['generations']['evolve_step_ms'], d['evolved'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches52.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_l=$?
