# time bench sections for several library builds: bash scripts/variants.sh v1 v2 ... (tmp_k1/<v>.so)
P=paper_2504_08339_b200/libflatneat_b200.so
cp $P /tmp/cur.so
for v in "$@"; do
  cp tmp_k1/$v.so $P
  for pop in random lineage; do python scripts/run_c5_distance.py 5 $pop | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v $pop', round(d['ms'],4), round(d['roofline']['frac'],4))"; done
done
cp /tmp/cur.so $P
