#!/bin/bash
# one compute-sanitizer tool per call: racecheck | synccheck | memcheck
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TOOL=${1:-racecheck}
EXTRA=""
[ "$TOOL" = "racecheck" ] && EXTRA="--racecheck-report all"
timeout 300 python tools/sanitize.py --quick > gpurun_out/r02_san_${TOOL}_plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/r02_san_${TOOL}_plain.log
timeout ${2:-1800} /usr/local/cuda/bin/compute-sanitizer --tool $TOOL $EXTRA --error-exitcode 9 \
   --print-limit 200 python tools/sanitize.py ${3:---quick} > gpurun_out/r02_san_${TOOL}.log 2>&1
echo "sanitizer rc=$?" >> gpurun_out/r02_san_${TOOL}.log
tail -5 gpurun_out/r02_san_${TOOL}.log
