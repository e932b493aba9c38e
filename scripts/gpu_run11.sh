python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench11.json 2>gpurun_out/bench11.err; echo bench=$?; python -c "import json;d=json.load(open('gpurun_out/bench11.json'));print(round(d['value']/1e9,2),'Gevals/s', d['kernels'], d['generations'])"; tail -3 gpurun_out/bench11.err
for k in k_mutate_apply k_transform k_forward; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 3 -c 1 -f -o gpurun_out/prof11_$k python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof11_$k.log 2>&1; echo ncu_$k=$?
done
