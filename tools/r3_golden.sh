timeout 900 python -m pytest tests/test_gpu_golden.py -q -m gpu -rxX 2>&1 | tail -6
timeout 600 python tools/c4_gate_svd.py tools/ab_libs/c4_thetas2.npz 2>&1 | tail -3
