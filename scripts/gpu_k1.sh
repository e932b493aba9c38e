python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform --launch-skip 4 -c 1 -f -o gpurun_out/prof_k1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu=$?
