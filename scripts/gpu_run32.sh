python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests/test_gpu_hyper.py tests/test_gpu_evolve.py -q -x > gpurun_out/pytest32.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest32.log
timeout 600 python bench.py --no-cpu-baseline --no-generations > gpurun_out/bench32.json 2>gpurun_out/bench32.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench32.json'));print(d['c4_hyperneat'], d['e2e'])"; tail -3 gpurun_out/bench32.err
