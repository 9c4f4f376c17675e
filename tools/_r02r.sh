set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02r_gpu_tests.log 2>&1; tail -2 gpurun_out/r02r_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; cat gpurun_out/r02r_smoke.log
timeout 900 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02r_ref.json 2> gpurun_out/r02r_ref.err
timeout 200 python tools/cipher_bench.py C1 C2 C3 C4 C5 > gpurun_out/r02r_cipher.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02r_launches.csv python bench.py --steps 2 --warmup 1 --frames 4 --no-configs --no-cpu-baseline --no-rows --clips 2 > gpurun_out/r02r_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prbg_chain_walk|k_prbg_verify_emit" -c 2 -o gpurun_out/r02r_full -f python tools/ncu_capture.py > gpurun_out/r02r_ncu_full.log 2>&1
tail -2 gpurun_out/r02r_ncu_full.log
timeout 300 python bench.py --shard-devices 0,0,0,0 --no-configs --no-rows --no-cpu-baseline > gpurun_out/r02r_shard4.json 2> gpurun_out/r02r_shard4.err
