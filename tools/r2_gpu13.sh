mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_queries.py tests/test_gpu_acceptance.py -q -m gpu -x > gpurun_out/r2_pytest13.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest13.log
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/r2_qr_case13.txt 2>&1
rm -rf /tmp/abrepo && cp -r . /tmp/abrepo && (cd /tmp/abrepo/paper_2601_04422_b200/csrc && make -s clean && make -s AB=1 -j16 > /dev/null 2>&1)
(cd /tmp/abrepo && REPS=1 MPSIM_QR_TRACE=1 timeout 300 python tools/qr_case.py > $GRAFT_REPO_ROOT/gpurun_out/r2_qr_trace13.txt 2>&1)
