# K3x ncu: one scatter round and one K3t round at C4 (--set full), and a launch list
CONFIG=C4 NF=2 CVE_B200_SCATTER=1 ncu --set full --clock-control none -k regex:scatter -s 2 -c 1 --csv --page raw --log-file gpurun_out/k3x_full_raw.csv python tools/fdec_probe.py > gpurun_out/k3x_ncu1.log 2>&1
CONFIG=C4 NF=2 ncu --set full --clock-control none -k regex:decrypt_round_tiles -s 2 -c 1 --csv --page raw --log-file gpurun_out/k3t_full_raw.csv python tools/fdec_probe.py > gpurun_out/k3x_ncu2.log 2>&1
CONFIG=C4 NF=2 CVE_B200_SCATTER=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decrypt|k_shift" --csv --log-file gpurun_out/k3x_launches.csv python tools/fdec_probe.py > /dev/null 2>&1
