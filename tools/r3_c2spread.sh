#!/bin/bash
timeout 600 python tools/c2_spread.py
timeout 600 python tools/c2_spread.py cx
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
echo "== A/B build MPSIM_GRAM3M=1"; MPSIM_GRAM3M=1 timeout 600 python tools/c2_spread.py
echo "== A/B build MPSIM_W32=1 (kW32MinN 512: C2 stays W16)"; MPSIM_QR=4 timeout 600 python tools/c2_spread.py
cp /tmp/product.so $L
