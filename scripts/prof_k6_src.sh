# ncu source page of K6 attrs at C5 (the working tree's build)
export FNB_STEP_GRAPH=0 FNB_GEN_GRAPH=0
T=${TAG:-k6}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mutate_attrs" --launch-skip 0 -c 1 -f -o gpurun_out/${T} python scripts/run_c5_generation.py 1 > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${T}_src.csv 2>/dev/null
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
rm -f gpurun_out/${T}.ncu-rep
