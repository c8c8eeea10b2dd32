#!/bin/bash
# DRAM traffic of one persistent sweep launch (64 gates, chi=512) per L2-hint policy (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum
for h in 0 2; do
  MPSIM_L2HINT=$h timeout 600 ncu --metrics $M --clock-control none -k regex:jacobi_sweep -s 3 -c 1 --csv env NGATES=64 python tools/ncu_case.py > gpurun_out/r3_ncu_l2_$h.csv 2>&1
  echo "== l2hint $h"; grep -E "dram__|gpu__time|lts__" gpurun_out/r3_ncu_l2_$h.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
cp /tmp/product.so $L
