timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-generations > gpurun_out/bq.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bq.json'));print(d['value'], d['kernels'])"
timeout 600 python scripts/run_c5_generation.py 4 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_transform --csv python scripts/run_c5_generation.py 2 2>/dev/null | grep k_transform | tail -2 | cut -c1-40,200-
