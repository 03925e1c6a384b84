#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bounds.py -x -q -p no:cacheprovider > gpurun_out/r02_bounds.log 2>&1
echo "bounds rc=$?" >> gpurun_out/r02_bounds.log
timeout 1500 python tools/race_stress.py 100 > gpurun_out/r02_race_stress.jsonl 2> gpurun_out/r02_race_stress.err
echo "race rc=$?" >> gpurun_out/r02_race_stress.err
bash tools/ncu_src.sh > gpurun_out/r02_ncu_src.out 2>&1
tail -2 gpurun_out/r02_bounds.log; tail -2 gpurun_out/r02_race_stress.err
