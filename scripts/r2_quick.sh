# quick GPU check: v6 parity subset + c5 apply/PCG bench (no stage leg, no CPU baseline)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_diag_small or configs_sampled or v6 or c5" > gpurun_out/r2_t.log 2>&1; tail -3 gpurun_out/r2_t.log
timeout 600 python bench.py --no-stage --no-cpu-baseline --steps 50 > gpurun_out/r2_b.json 2> gpurun_out/r2_b.err
python -c "
import json; d=json.load(open('gpurun_out/r2_b.json'))
print('apply ms %.4f GDOF/s %.1f frac %.3f  CG it/s %.0f iters %s clocks %s' % (d['roofline']['launch_ms'], d['value'], d['roofline']['frac'], d['pcg']['iters_per_s'], d['pcg']['iters'], d['clocks']))"
tail -3 gpurun_out/r2_b.err
