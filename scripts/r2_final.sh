# what the driver runs at round end: GPU tests, smoke, default bench, reference arm
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2f_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; tail -2 gpurun_out/r2f_smoke.log
timeout 1500 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo bench rc=$?; tail -c 300 gpurun_out/r2f_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2f_ref.json 2> gpurun_out/r2f_ref.err; echo ref rc=$?; tail -c 300 gpurun_out/r2f_ref.json
