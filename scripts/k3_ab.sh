# K3 A/B: lane-per-genome (default) vs warp-per-genome (FNB_K3=warp)
timeout 900 python -m pytest tests -m gpu -q -x -k "distance or evolve or species or generation" 2>&1 | tail -2
FNB_K3=warp timeout 900 python -m pytest tests -m gpu -q -x -k "distance" 2>&1 | tail -1
for mode in lane warp lane; do for pop in random lineage; do FNB_K3=$mode python scripts/run_c5_distance.py 5 $pop | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$mode $pop', round(d['ms'],4), round(d['roofline']['frac'],4))"; done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof_k3l python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
ncu -i gpurun_out/prof_k3l.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_k3l_src.csv 2>/dev/null
