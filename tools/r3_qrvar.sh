REPS=8 timeout 300 python tools/qr_case.py 2>&1 | tail -8
nproc; uptime
REPS=4 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3_qrvar_ncu.csv python tools/qr_case.py > gpurun_out/r3_qrvar_ncu.log 2>&1
tail -4 gpurun_out/r3_qrvar_ncu.log
