python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 600 python -m pytest tests/test_gpu_forward.py -q -x > gpurun_out/pytest22.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest22.log
timeout 300 python bench.py --no-cpu-baseline --no-c5 --no-generations > gpurun_out/bench22.json 2>gpurun_out/bench22.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench22.json'));print(d['value']/1e9, d['e2e'], d['kernels'])"; tail -3 gpurun_out/bench22.err
