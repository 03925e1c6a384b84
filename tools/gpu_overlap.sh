python -m paper_2604_11558_b200.build > /dev/null
python tools/overlap_probe.py base
python tools/overlap_probe.py free
CURVIGPU_GEMM_CPS=1 CURVIGPU_FRONT_CPS=1 python tools/overlap_probe.py serial
CURVIGPU_GEMM_CPS=1 CURVIGPU_FRONT_CPS=1 python tools/overlap_probe.py free
CURVIGPU_GEMM_CPS=1 CURVIGPU_FRONT_CPS=1 python tools/overlap_probe.py split
CURVIGPU_GEMM_CPS=1 python tools/overlap_probe.py split
CURVIGPU_FRONT_CPS=1 python tools/overlap_probe.py split
CURVIGPU_FRONT_CPS=1 python tools/overlap_probe.py free
THETA=fft python tools/profile_step.py > gpurun_out/plain_step_fft.log 2>&1 && \
THETA=fft timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|theta_|fbuild|disk_ftheta" -s 2 -c 4 \
     -o gpurun_out/prof_step_fft python tools/profile_step.py > gpurun_out/ncu_step_fft.log 2>&1; echo "ncu fft rc=$?"
