set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02s_gpu_tests.log 2>&1; tail -2 gpurun_out/r02s_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; cat gpurun_out/r02s_smoke.log
timeout 900 python bench.py > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s_ref.json 2> gpurun_out/r02s_ref.err
L=gpurun_out/r02s_wide_sweep.log; : > $L
for s in 41 42 43; do timeout 900 python tools/wide_sweep.py $s 90 700 9 >> $L 2>&1; done
grep -E "failures|FAIL|EXC" $L
