#!/bin/bash
# round-2 first GPU pass: full GPU test suite, a short bench line, the
# sanitizer workload once without instrumentation
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_tests.log
timeout 300 python tools/sanitize.py > gpurun_out/r02_sanitize_plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/r02_sanitize_plain.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
echo "bench rc=$?" >> gpurun_out/r02_bench.err
tail -3 gpurun_out/r02_tests.log
