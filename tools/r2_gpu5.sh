mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_chi_cap.py tests/test_gpu_queries.py -q -m gpu > gpurun_out/r2_pytest5.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest5.log
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qrp_panel_cluster -s 40 -c 1 -o gpurun_out/r2_qrpanel python tools/qr_case.py > gpurun_out/r2_qrpanel_ncu.log 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:qrp_update_kernel -s 40 -c 1 -o gpurun_out/r2_qrupd python tools/qr_case.py > gpurun_out/r2_qrupd_ncu.log 2>&1
TOOL=memcheck bash tools/r2_sanitize.sh
