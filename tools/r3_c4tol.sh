L=paper_2601_04422_b200/libmpsim_gpu.so
cp tools/ab_libs/jtol.so $L
for v in "MPSIM_JTOL=4" "MPSIM_JTOL=1" "MPSIM_JTOL=0.25" "MPSIM_JTOL=1 MPSIM_QR=0" "MPSIM_JTOL=4 MPSIM_QR=0"; do
 echo "== $v"; env $v timeout 900 python -m pytest tests/test_gpu_golden.py::test_c4_window_reaching_chi1024_against_fixture -q -m gpu 2>&1 | grep -E "^E  +AssertionError|passed|failed" | head -2
done
