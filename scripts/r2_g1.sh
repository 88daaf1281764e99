set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_diag_small or configs_sampled or v6 or c5 or apply_configs_full" > gpurun_out/r2_t1.log 2>&1; tail -5 gpurun_out/r2_t1.log
timeout 600 python bench.py --no-stage --no-cpu-baseline --steps 50 > gpurun_out/r2_b1.json 2> gpurun_out/r2_b1.err; tail -c 1500 gpurun_out/r2_b1.json; tail -3 gpurun_out/r2_b1.err
