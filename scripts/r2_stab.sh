timeout 1200 python -m pytest tests/test_gpu_stab.py -x -q > gpurun_out/r2_stab.log 2>&1; tail -30 gpurun_out/r2_stab.log
timeout 1500 python tools/tg_eoc.py > gpurun_out/r2_tg.log 2>&1; cat gpurun_out/r2_tg.log | tail -20
