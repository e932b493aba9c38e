set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
for s in 1 2 4; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --spt $s > gpurun_out/bench_spt$s.json 2>gpurun_out/bench_spt$s.err; echo spt$s=$?; python -c "import json;d=json.load(open('gpurun_out/bench_spt$s.json'));print('spt',$s,d['value']/1e9,'Gevals/s', d['kernels'], d['roofline']['frac'], d['roofline']['smem']['frac'])"; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 2 -c 1 -o gpurun_out/prof_forward2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1; echo ncu=$?
