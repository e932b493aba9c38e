timeout 1200 python -m pytest tests/test_gpu_evolve.py -q -x > gpurun_out/pytest_evolve.log 2>&1; echo pytest=$?; tail -60 gpurun_out/pytest_evolve.log
