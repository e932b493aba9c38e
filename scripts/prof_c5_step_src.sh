cd $GRAFT_REPO_ROOT
export FNB_STEP_GRAPH=0 FNB_GEN_GRAPH=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_mutate_attrs|k_transform" --launch-skip 0 -c 2 -f -o gpurun_out/s3_c5 python scripts/run_c5_generation.py 1 > gpurun_out/s3_c5.log 2>&1; echo ncu=$?
for k in k_mutate_attrs k_transform; do
  ncu -i gpurun_out/s3_c5.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > gpurun_out/s3_src_$k.csv 2>/dev/null
  ncu -i gpurun_out/s3_c5.ncu-rep -k regex:$k --page raw --csv > gpurun_out/s3_raw_$k.csv 2>/dev/null
done
ls -la gpurun_out/
