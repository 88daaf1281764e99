timeout 1500 python -m pytest tests -m gpu -x -q -k "pcg or solve or halo or stage or rk or schwarz or visc or diag" > gpurun_out/r2_pcgt.log 2>&1; tail -3 gpurun_out/r2_pcgt.log
python tools/one_solve.py > gpurun_out/os.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/os_launches.csv python tools/one_solve.py > gpurun_out/os_ncu.log 2>&1; tail -1 gpurun_out/os.log
timeout 600 python bench.py --no-stage --no-cpu-baseline --no-configs --no-traffic --steps 50 > gpurun_out/r2_b.json 2> gpurun_out/r2_b.err
python -c "
import json; d=json.load(open('gpurun_out/r2_b.json'))
print('apply ms %.4f GDOF/s %.1f frac %.3f  CG it/s %.0f iters %s ms %.2f' % (d['roofline']['launch_ms'], d['value'], d['roofline']['frac'], d['pcg']['iters_per_s'], d['pcg']['iters'], d['pcg']['ms_per_solve']))"
