# quick bench of the current build (P=5 only builds are fine): default path, then v4
set -x
timeout 300 python bench.py --no-cpu-baseline --solves 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json; python -c "import json;d=json.load(open('gpurun_out/bench.json'));print('apply ms',d['ms_per_step'],'frac',d['roofline']['frac'],'pcg it/s',d['pcg']['iters_per_s'])"; tail -3 gpurun_out/bench.err
