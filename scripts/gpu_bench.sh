# quick bench of the current build (P=5-only builds are fine)
timeout 300 python bench.py --no-cpu-baseline --no-stage --solves 2 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('apply ms',d['ms_per_step'],'frac',d['roofline']['frac'],'pcg it/s',d['pcg']['iters_per_s'])"
tail -3 gpurun_out/bench.err
