# K3 parity tests + C5 distance timing + one ncu capture
timeout 900 python -m pytest tests -m gpu -q -x -k "distance or evolve or generation or species" 2>&1 | tail -2
for pop in random lineage; do python scripts/run_c5_distance.py 5 $pop | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$pop', d['ms'], d['roofline']['frac'])"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof_k3b python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
ncu -i gpurun_out/prof_k3b.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_k3b_src.csv 2>/dev/null
