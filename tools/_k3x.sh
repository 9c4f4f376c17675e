# K3x (scatter-form inverse round): tests, then cipher_bench decrypt vs K3t
timeout 300 python -m pytest tests/test_round_kernels.py -x -q -k k3x 2>&1 | tail -15
python tools/cipher_bench.py C1 C3 C4 C5
for T in 4 8 16; do echo "T=$T"; CVE_B200_SCATTER=1 CVE_B200_SCATTER_T=$T python tools/cipher_bench.py C1 C3 C4 C5; done
