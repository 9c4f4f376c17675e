# K3f vs K3t launch lists (tools/fdec_probe.py under ncu)
set -x
for C in C4 C5; do
  CONFIG=$C python tools/fdec_probe.py
  CONFIG=$C CVE_B200_FDEC=1 python tools/fdec_probe.py
  CONFIG=$C ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decrypt|inv_diff|k_shift" --csv --log-file gpurun_out/fdec_base_$C.csv python tools/fdec_probe.py > /dev/null 2>&1
  CONFIG=$C CVE_B200_FDEC=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decrypt|inv_diff|k_shift" --csv --log-file gpurun_out/fdec_k3f_$C.csv python tools/fdec_probe.py > /dev/null 2>&1
done
