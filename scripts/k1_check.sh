set -x
P=paper_2504_08339_b200/libflatneat_b200.so
cp $P /tmp/new.so; cp tmp_k1/old.so $P
python scripts/k1_dump.py gpurun_out/k1_old.npz 2>&1 | tail -3
cp /tmp/new.so $P
python scripts/k1_dump.py gpurun_out/k1_new.npz 2>&1 | tail -3
python scripts/k1_dump.py cmp gpurun_out/k1_old.npz gpurun_out/k1_new.npz; rm -f gpurun_out/*.npz
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py --no-cpu-baseline --no-c5 --no-generations > gpurun_out/bq.json 2>gpurun_out/bq.err; tail -2 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print(d['kernels'], d['value'])"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform --launch-skip 2 -c 1 -f -o gpurun_out/prof_k1b python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k1=$?
ncu -i gpurun_out/prof_k1b.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof_k1b_src.csv 2>/dev/null
