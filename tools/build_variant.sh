#!/bin/bash
# Builds a product-configuration variant of the library out of tree with extra nvcc flags:
#   tools/build_variant.sh <name> "<EXTRA nvcc flags>"  ->  tools/ab_libs/<name>.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/mpsim_var_$1
rm -rf $T; mkdir -p $T/pkg/csrc $T/include tools/ab_libs
cp "$R"/paper_2601_04422_b200/csrc/*.cu* "$R"/paper_2601_04422_b200/csrc/*.h "$R"/paper_2601_04422_b200/csrc/*.cpp "$R"/paper_2601_04422_b200/csrc/Makefile $T/pkg/csrc/
cp -r "$R"/include/. $T/include/
make -C $T/pkg/csrc EXTRA="$2" -j8 > $T/make.log 2>&1 || (grep -B2 -A5 error $T/make.log | head -30; false)
cp $T/pkg/libmpsim_gpu.so "$R/tools/ab_libs/$1.so"
grep -A2 "19jacobi_sweep_kernel\|jacobi_sweep_w32_kernel" $T/pkg/csrc/build/jacobi_split.ptxas.log $T/pkg/csrc/build/jacobi_w32.ptxas.log | grep -E "spill|Used" | head -4
echo built tools/ab_libs/$1.so
