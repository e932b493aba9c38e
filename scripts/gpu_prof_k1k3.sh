# ncu --set full captures of K1 (transform at C2) and K3 (distance at C5), with source pages
python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform --launch-skip 2 -c 1 -f -o gpurun_out/prof_k1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof_k3 python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
for r in prof_k1 prof_k3; do
  ncu -i gpurun_out/$r.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${r}_src.csv 2>/dev/null
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ls -la gpurun_out
