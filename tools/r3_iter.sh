#!/bin/bash
# Round-3 dev loop: parity subset on the product build, sweep profile, then
# A/B of the cluster-sweep knobs on the A/B build (tools/ab_libs/ab.so).
mkdir -p gpurun_out
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
if [ "${SKIP_TESTS:-0}" != 1 ]; then
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_svd.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py} -x -q -m gpu 2>&1 | tail -4
fi
MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -13
cp tools/ab_libs/ab.so $L
for v in ${VARIANTS:-"MPSIM_SWEEP_CL=0" "MPSIM_GROUP=4" "MPSIM_GROUP=6" "MPSIM_GROUP=8" "MPSIM_GROUP=12"}; do
  echo "== $v"; env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2
done
cp /tmp/product.so $L
