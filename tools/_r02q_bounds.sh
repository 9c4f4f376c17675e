set -x
mkdir -p gpurun_out
export CVE_B200_LIBRARY=$PWD/tools/variants/lib_bounds.so
timeout 1800 python -m pytest tests -m gpu -q -k "not c_caller" > gpurun_out/r02q_bounds_tests.log 2>&1; tail -3 gpurun_out/r02q_bounds_tests.log
L=gpurun_out/r02q_bounds_sweep.log; : > $L
for s in 31 32; do timeout 900 python tools/wide_sweep.py $s 90 700 9 >> $L 2>&1; done
CVE_B200_NO_ROWS=1 timeout 600 python tools/wide_sweep.py 33 60 600 12 >> $L 2>&1
CVE_B200_ROWS_DECRYPT=1 timeout 600 python tools/wide_sweep.py 34 60 600 12 >> $L 2>&1
CVE_B200_NO_TILES=1 timeout 600 python tools/wide_sweep.py 35 60 600 12 >> $L 2>&1
timeout 900 python tools/large_side_check.py 4096,256,2 5000,8,1 4100,1025,1 >> $L 2>&1
grep -E "failures|FAIL|EXC" $L
