python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.json 2>gpurun_out/bench13.err; python -c "import json;d=json.load(open('gpurun_out/bench13.json'));print(round(d['value']/1e9,2),'Gevals/s', d['kernels'], d['generations'])"; tail -3 gpurun_out/bench13.err
for spec in "k_mutate_apply 3" "k_transform 3" "k_forward 4"; do set -- $spec
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip $2 -c 1 -f -o gpurun_out/prof13_$1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof13_$1.log 2>&1; echo ncu_$1=$?
done
