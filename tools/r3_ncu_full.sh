#!/bin/bash
# ncu --set full of one persistent sweep launch (64 gates, chi=512), product build.
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-jacobi_sweep} -s ${SKIP:-3} -c 1 -o gpurun_out/${OUT:-r3_sweep} -f env NGATES=64 python tools/ncu_case.py > gpurun_out/${OUT:-r3_sweep}.log 2>&1
tail -3 gpurun_out/${OUT:-r3_sweep}.log
