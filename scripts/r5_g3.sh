# default build after the pitched-plane experiment (DG_V6_PITCH 0): identical time / checksum to HEAD, parity, ncu of the stage applies
DG_LIBRARY=$PWD/build_ab/libH2.so timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn | tail -1; timeout 300 python tools/ab_apply.py 2>&1 | grep -v Warn | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py -q -x 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)6' -s 30 -c 1 -o gpurun_out/r5_apply6_p6 python tools/stage_one.py > gpurun_out/r5_apply6_p6.log 2>&1; echo "p6 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_apply6<\(int\)7, \(bool\)0, \(int\)3' -s 10 -c 1 -o gpurun_out/r5_apply6_p7 python tools/stage_one.py > gpurun_out/r5_apply6_p7.log 2>&1; echo "p7 rc=$?"
