timeout 1800 python -m pytest tests -m gpu -x -q -k "pcg or stage or rk or schwarz or visc or smoke or solve" > gpurun_out/r2g_t.log 2>&1; tail -3 gpurun_out/r2g_t.log
timeout 900 python bench.py --no-cpu-baseline --no-traffic --steps 30 > gpurun_out/r2g_b.json 2> gpurun_out/r2g_b.err; echo rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2g_b.json').read().splitlines()[-1])
print('apply', d['roofline']['launch_ms'], 'pcg', d['pcg']['iters_per_s'], 'stage', d['stage']['ms_per_stage'], 'rk', d['stage']['rk_step']['ms_per_step'], 'vv', d['stage']['vv_step']['ms_per_step'], 'launches', d['gpu_launches'])
for k,v in d['configs'].items(): print(k, 'helm', v['helmholtz'], v.get('poisson_P6'))
print('halo', d['halo'])
PY
