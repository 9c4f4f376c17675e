# K3f chunk-height / thread sweep (tools/fdec_probe.py, in-product times)
for C in C4 C5 C3; do
  CONFIG=$C python tools/fdec_probe.py
  for cr in 16 15 10 8 6 5 4 3; do for th in 256 512; do
    echo -n "cr=$cr th=$th  "; CONFIG=$C CVE_B200_FDEC=1 CVE_B200_FDEC_CR=$cr CVE_B200_FDEC_THREADS=$th python tools/fdec_probe.py
  done; done
done
