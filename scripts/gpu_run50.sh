python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_evolve.py -q -x > gpurun_out/pytest50.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest50.log
timeout 300 python scripts/run_c5_distance.py 5 > gpurun_out/c5_50.json 2>&1; echo c5=$?; python -c "import json;d=json.load(open('gpurun_out/c5_50.json'));print(d['ms'], d['roofline']['frac'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof50_k3 python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu=$?
