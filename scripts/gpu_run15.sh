python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/bench15.json 2>gpurun_out/bench15.err; python -c "import json;d=json.load(open('gpurun_out/bench15.json'));print(round(d['value']/1e9,2),'Gevals/s', d['kernels'], d['generations'])"; tail -3 gpurun_out/bench15.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches15.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?
