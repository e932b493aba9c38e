# A round's GPU evidence: full bench line, launch list, ncu summaries; compute-sanitizer memcheck + racecheck of key tests
python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python bench.py > gpurun_out/bench${TAG:-r01d}.json 2>gpurun_out/bench${TAG:-r01d}.err; echo bench=$?; tail -2 gpurun_out/bench${TAG:-r01d}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches${TAG:-r01d}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_forward --launch-skip 5 -c 1 -f -o gpurun_out/prof${TAG:-r01d}_k2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof${TAG:-r01d}_k3_c5 python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hyper_rollout -c 1 -f -o gpurun_out/prof${TAG:-r01d}_c4 python -c "
import torch,bench
dev=torch.device('cuda',0); fl=torch.empty(256<<20,dtype=torch.uint8,device=dev)
bench.c4_hyperneat(dev, torch.cuda.current_stream(), fl, reps=1)" > /dev/null 2>&1; echo ncu_c4=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_mutate_attrs|k_mutate_apply|k_crossover" --launch-skip 9 -c 3 -f -o gpurun_out/prof${TAG:-r01d}_step python scripts/run_c2_generation.py 6 > /dev/null 2>&1; echo ncu_step=$?
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_ops.py tests/test_gpu_hyper.py tests/test_gpu_forward.py -q -x -k "not c2_shape" > gpurun_out/memcheck${TAG:-r01d}.log 2>&1; echo memcheck=$?; tail -4 gpurun_out/memcheck${TAG:-r01d}.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 3 python -m pytest tests/test_gpu_ops.py -q -x -k "distance" > gpurun_out/racecheck${TAG:-r01d}.log 2>&1; echo racecheck=$?; tail -4 gpurun_out/racecheck${TAG:-r01d}.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_evolve.py -q -x -k "split_step or generation_loop" > gpurun_out/memcheck${TAG:-r01d}b.log 2>&1; echo memcheck_evolve=$?; tail -4 gpurun_out/memcheck${TAG:-r01d}b.log
