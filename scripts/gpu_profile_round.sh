# A round's GPU evidence: full bench line, launch list, ncu summaries; compute-sanitizer memcheck + racecheck of key tests
# (ncu cannot profile kernel nodes of graphs with conditional nodes, and its replay of the evaluate graph's
# k_forward node fails with LaunchFailed (round 2): the launch list runs eagerly, FNB_GEN_GRAPH=0 FNB_STEP_GRAPH=0)
T=${TAG:-r02}
python -c "import paper_2504_08339_b200" 2>/dev/null || { echo "library stale: rebuilding"; python -c "import __graft_entry__ as g; g.build()"; }
timeout 900 python bench.py > gpurun_out/bench$T.json 2>gpurun_out/bench$T.err; echo bench=$?; tail -2 gpurun_out/bench$T.err
FNB_GEN_GRAPH=0 FNB_STEP_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches$T.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo ncu_l=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_forward --launch-skip 5 -c 1 -f -o gpurun_out/prof${T}_k2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k2=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_transform --launch-skip 5 -c 1 -f -o gpurun_out/prof${T}_k1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5 --no-generations > /dev/null 2>&1; echo ncu_k1=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_distance --launch-skip 2 -c 1 -f -o gpurun_out/prof${T}_k3_c5 python scripts/run_c5_distance.py 1 > /dev/null 2>&1; echo ncu_k3=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_hyper_rollout -c 1 -f -o gpurun_out/prof${T}_c4 python -c "
import torch,bench
dev=torch.device('cuda',0); fl=torch.empty(256<<20,dtype=torch.uint8,device=dev)
bench.c4_hyperneat(dev, torch.cuda.current_stream(), fl, reps=1)" > /dev/null 2>&1; echo ncu_c4=$?
FNB_STEP_GRAPH=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_mutate_attrs|k_mutate_apply|k_crossover" --launch-skip 9 -c 3 -f -o gpurun_out/prof${T}_step python scripts/run_c2_generation.py 6 > /dev/null 2>&1; echo ncu_step=$?
FNB_STEP_GRAPH=0 timeout 900 ncu --set full --clock-control none -k regex:"k_mutate_attrs|k_mutate_apply|k_crossover|k_transform" --launch-skip 0 -c 4 -f -o gpurun_out/prof${T}_c5step python scripts/run_c5_generation.py 1 > /dev/null 2>&1; echo ncu_c5step=$?
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_ops.py tests/test_gpu_hyper.py tests/test_gpu_forward.py tests/test_gpu_boundary.py tests/test_gpu_packed.py -q -x -k "not c2_shape and not 1e8 and not full_grid" > gpurun_out/memcheck$T.log 2>&1; echo memcheck=$?; tail -4 gpurun_out/memcheck$T.log
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 3 python -m pytest tests/test_gpu_ops.py -q -x -k "distance" > gpurun_out/racecheck$T.log 2>&1; echo racecheck=$?; tail -4 gpurun_out/racecheck$T.log
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 3 python -m pytest tests/test_gpu_evolve.py tests/test_evolve_run.py tests/test_gpu_sharded.py -q -x -k "split_step or generation_loop_bit_exact[ or run_equals or world1" > gpurun_out/memcheck${T}b.log 2>&1; echo memcheck_evolve=$?; tail -4 gpurun_out/memcheck${T}b.log
