timeout 1200 python -m pytest tests/test_gpu_halo.py -x -q > gpurun_out/r2_halo.log 2>&1; tail -30 gpurun_out/r2_halo.log
timeout 600 python bench.py --no-stage --no-cpu-baseline --steps 50 > gpurun_out/r2_b.json 2> gpurun_out/r2_b.err
python -c "
import json; d=json.load(open('gpurun_out/r2_b.json'))
print('apply ms %.4f GDOF/s %.1f frac %.3f  CG it/s %.0f iters %s clocks %s' % (d['roofline']['launch_ms'], d['value'], d['roofline']['frac'], d['pcg']['iters_per_s'], d['pcg']['iters'], d['clocks']))"
