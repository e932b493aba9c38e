# generation-loop parity tests + the C2/C5 generation numbers
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bg.json 2>gpurun_out/bg.err; tail -2 gpurun_out/bg.err
python - <<'PY'
import json;d=json.load(open('gpurun_out/bg.json'))
print('value', d['value'], d['kernels'])
print('gen', d['generations']['ms_per_generation'], d['generations']['evaluate_ms'], d['generations']['evolve_step_ms'])
print('c5gen', d['c5_generation']['ms_per_generation'], d['c5_generation']['evaluate_ms'], d['c5_generation']['evolve_step_ms'])
print('c5dist', d['c5_distance']['ms'], d['c5_distance_lineage']['ms'])
PY
