#!/bin/bash
# Builds the A/B-knob variant of the library (make AB=1) out of tree into tools/ab_libs/ab.so.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/mpsim_ab_build
mkdir -p $T/pkg $T/include tools/ab_libs
rm -rf $T/pkg/csrc; mkdir -p $T/pkg/csrc; cp "$R"/paper_2601_04422_b200/csrc/*.cu* "$R"/paper_2601_04422_b200/csrc/*.h "$R"/paper_2601_04422_b200/csrc/*.cpp "$R"/paper_2601_04422_b200/csrc/Makefile $T/pkg/csrc/
cp -r "$R"/include/. $T/include/
make -C $T/pkg/csrc AB=1 -j8 > $T/make.log 2>&1 || (tail -30 $T/make.log; false)
cp $T/pkg/libmpsim_gpu.so "$R/tools/ab_libs/ab.so"
echo built tools/ab_libs/ab.so
