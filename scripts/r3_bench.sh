# default bench (the driver's command) + launch list of the same command
timeout 1500 python bench.py > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err; echo rc=$?
python - <<'PY'
import json
d=json.load(open('gpurun_out/r3_bench.json'))
r=d['roofline']; print('apply', r['launch_ms'], 'GDOF/s', d['value'], 'frac', r['frac'], 'traffic', r['traffic'], r.get('traffic_over_algorithmic'), r['kernel'])
print('pcg', d['pcg']['iters_per_s'], d['pcg']['iters'], d['pcg']['ms_per_solve'])
print('stage', d['stage']['ms_per_stage'], d['stage']['pressure_iters'], d['stage']['velocity_iters'], 'stab', d['stage']['div_stab'], 'rk', d['stage']['rk_step']['ms_per_step'], 'vv', d['stage']['vv_step']['ms_per_step'])
print('halo', d['halo'])
for k,v in d['configs'].items(): print(k, {kk: vv for kk, vv in v.items() if kk != 'workload'})
print('e2e', d['e2e'], 'clocks', d['clocks'], 'launches', d['gpu_launches'])
print('cpu', d['cpu_baseline'])
PY
tail -5 gpurun_out/r3_bench.err
