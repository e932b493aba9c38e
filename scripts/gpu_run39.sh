python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python -m pytest tests/test_gpu_hyper.py -q -x > gpurun_out/pytest39.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest39.log
timeout 600 python -c "
import json,torch,bench
dev=torch.device('cuda',0); fl=torch.empty(256<<20,dtype=torch.uint8,device=dev)
print(json.dumps(bench.c4_hyperneat(dev, torch.cuda.current_stream(), fl, reps=5)))"
