timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench7.json'));print(json.dumps(d, indent=1))" | head -80; tail -3 gpurun_out/bench7.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu=$?
