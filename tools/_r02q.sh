set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02q_gpu_tests.log 2>&1; tail -2 gpurun_out/r02q_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; cat gpurun_out/r02q_smoke.log
timeout 900 python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02q_ref.json 2> gpurun_out/r02q_ref.err
