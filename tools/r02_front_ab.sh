#!/bin/bash
# A/B of fused-front builds on config 5: kernel times per library variant
#   VARIANTS="label:lib[:ENV=V,ENV=V] ..." bash tools/r02_front_ab.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
OUT=gpurun_out/r02_front_ab.txt
: > $OUT
for rep in 1 2; do
for v in $VARIANTS; do
  IFS=: read label lib envs <<< "$v"
  echo "== $label ($lib $envs)" >> $OUT
  env CURVIGPU_LIB=$PWD/paper_2604_11558_b200/$lib CONFIGS=${CONFIGS:-5} $(echo $envs | tr ',' ' ') timeout 600 python tools/kernel_times.py >> $OUT 2>&1
done
done
if [ -n "$TESTLIB" ]; then
CURVIGPU_LIB=$PWD/paper_2604_11558_b200/$TESTLIB timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r02_front_ab_tests.log 2>&1
echo "tests($TESTLIB) rc=$?" >> $OUT
fi
cat $OUT
