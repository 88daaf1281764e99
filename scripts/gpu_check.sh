# parity tests + bench (current default path) + bench with the v4 apply for comparison
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
DG_APPLY_IMPL=v4 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_v4.json 2>&1; cat gpurun_out/bench_v4.json | cut -c1-300
