python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest34.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest34.log
timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-generations > gpurun_out/bench34.json 2>gpurun_out/bench34.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench34.json'));print(d['value']/1e9, d['e2e']['value']/1e9, d['kernels'], d['roofline']['frac'])"; tail -3 gpurun_out/bench34.err
timeout 900 python scripts/sweep_forward.py > gpurun_out/sweep34.json 2>&1; echo sweep=$?; head -c 1500 gpurun_out/sweep34.json
