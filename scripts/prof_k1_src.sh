# ncu source pages of K1 at C2 (bench shapes) and C5 (generation driver)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform --launch-skip 5 -c 1 -f -o gpurun_out/k1c2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_c2=$?
FNB_STEP_GRAPH=0 FNB_GEN_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform -c 1 -f -o gpurun_out/k1c5 python scripts/run_c5_generation.py 1 > /dev/null 2>&1; echo ncu_c5=$?
for t in k1c2 k1c5; do
  ncu -i gpurun_out/$t.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${t}_src.csv 2>/dev/null
  ncu -i gpurun_out/$t.ncu-rep --page raw --csv > gpurun_out/${t}_raw.csv 2>/dev/null
  rm -f gpurun_out/$t.ncu-rep
done
