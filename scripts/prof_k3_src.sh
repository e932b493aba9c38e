# ncu source page of k_distance at C5 (random and lineage populations)
for pop in random lineage; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/k3_$pop python scripts/run_c5_distance.py 1 $pop > /dev/null 2>&1; echo ncu_$pop=$?
  ncu -i gpurun_out/k3_$pop.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k3_${pop}_src.csv 2>/dev/null
  ncu -i gpurun_out/k3_$pop.ncu-rep --page raw --csv > gpurun_out/k3_${pop}_raw.csv 2>/dev/null
  rm -f gpurun_out/k3_$pop.ncu-rep
done
