mkdir -p gpurun_out
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:site_qr_factor -s 30 -c 1 -o gpurun_out/r2_siteqr python tools/qr_case.py > gpurun_out/r2_siteqr_ncu.log 2>&1
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:site_qr_q -s 30 -c 1 -o gpurun_out/r2_siteqrq python tools/qr_case.py > gpurun_out/r2_siteqrq_ncu.log 2>&1
