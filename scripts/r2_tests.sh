# full GPU test suite with per-test durations
nproc
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2_pytest_gpu.log 2>&1; tail -40 gpurun_out/r2_pytest_gpu.log
