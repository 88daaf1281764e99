# pitched z planes in the n = 6 v6 slots (y-pass bank conflicts): A/B against HEAD (libH2), parity, PCG time
for i in 1 2; do DG_LIBRARY=$PWD/build_ab/libH2.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn | tail -1; timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -q -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "apply_every_element or pcg_c5" 2>&1 | tail -2
DG_LIBRARY=$PWD/build_ab/libH2.so timeout 300 python tools/pcg_breakdown.py 5 2>&1 | grep -v Warn | tail -2
timeout 300 python tools/pcg_breakdown.py 5 2>&1 | grep -v Warn | tail -2
# ncu of the P = 6 pressure apply and the P = 7 velocity apply inside a config-4 stage
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)6' -s 30 -c 1 -o gpurun_out/r5_apply6_p6 python tools/stage_one.py > gpurun_out/r5_apply6_p6.log 2>&1; echo "p6 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)7, \(bool\)0, \(int\)3' -s 10 -c 1 -o gpurun_out/r5_apply6_p7 python tools/stage_one.py > gpurun_out/r5_apply6_p7.log 2>&1; echo "p7 rc=$?"
