timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -40 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2>gpurun_out/bench5.err; python -c "import json;d=json.load(open('gpurun_out/bench5.json'));print(round(d['value']/1e9,2),'Gevals/s', d['kernels'])"
