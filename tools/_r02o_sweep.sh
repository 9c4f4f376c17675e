set -x
mkdir -p gpurun_out
L=gpurun_out/r02o_wide_sweep.log
: > $L
for s in 11 12 13 14; do timeout 900 python tools/wide_sweep.py $s 90 700 9 >> $L 2>&1; done
CVE_B200_NO_ROWS=1 timeout 600 python tools/wide_sweep.py 21 60 600 12 >> $L 2>&1
CVE_B200_ROWS_DECRYPT=1 timeout 600 python tools/wide_sweep.py 22 60 600 12 >> $L 2>&1
CVE_B200_NO_TILES=1 timeout 600 python tools/wide_sweep.py 23 60 600 12 >> $L 2>&1
CVE_B200_ROWS_PERSIST=1 timeout 600 python tools/wide_sweep.py 24 60 600 12 >> $L 2>&1
grep -c FAIL $L; grep "failures" $L
