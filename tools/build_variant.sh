#!/bin/bash
# A/B library variant: tools/build_variant.sh <label> [-DFLAG ...]  -> paper_2604_11558_b200/libcurvigpu_<label>.so
# (plan.cu recompiled with the extra flags, linked with the default build's setup.o / rng.o)
set -e
cd "$(dirname "$0")/.."
L=$1; shift
P=paper_2604_11558_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
  -Iinclude "$@" -c -o $P/build/plan_$L.o $P/csrc/plan.cu 2> $P/build/plan_$L.log
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libcurvigpu_$L.so $P/build/plan_$L.o $P/build/setup.o $P/build/rng.o
echo built $P/libcurvigpu_$L.so
