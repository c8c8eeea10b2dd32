L=paper_2601_04422_b200/libmpsim_gpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_svd.py -x -q -m gpu 2>&1 | tail -3
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -22
for v in MPSIM_EVD32_MAXOFF=0 MPSIM_EVD32_MAXOFF=1e-2 MPSIM_EVD32_MAXOFF=0 MPSIM_EVD32_MAXOFF=1e-2; do echo "== $v"; env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2; done
cp /tmp/product.so $L
