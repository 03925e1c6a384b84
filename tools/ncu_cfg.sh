#!/bin/bash
# ncu --set full with source correlation of one BASELINE config's step kernels:
#   CONFIG=4 THETA=fft bash tools/ncu_cfg.sh   -> gpurun_out/prof_c${CONFIG}_${THETA}.ncu-rep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
CONFIG=${CONFIG:-4}; THETA=${THETA:-fft}
CONFIG=$CONFIG THETA=$THETA python tools/profile_step.py > gpurun_out/plain_step_c$CONFIG.log 2>&1; echo "plain rc=$?"
CONFIG=$CONFIG THETA=$THETA timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"gemm_f64|theta_fast|fbuild|disk_ftheta|disk_step" -s ${SKIP:-4} -c ${COUNT:-4} \
   -f -o gpurun_out/prof_c${CONFIG}_${THETA} python tools/profile_step.py > gpurun_out/ncu_c$CONFIG.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_c$CONFIG.log
