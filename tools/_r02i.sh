set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
tail -c 400 gpurun_out/r02i_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02i_ref.json 2> gpurun_out/r02i_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02i_launches.csv python bench.py --steps 2 --warmup 1 --frames 4 --no-configs --no-cpu-baseline --no-rows --clips 2 > gpurun_out/r02i_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_encrypt_round_rows|k_decrypt_round_tiles|k_prbg_verify_emit" -c 3 -o gpurun_out/r02i_full -f python tools/ncu_capture.py > gpurun_out/r02i_ncu_full.log 2>&1
tail -2 gpurun_out/r02i_ncu_full.log
