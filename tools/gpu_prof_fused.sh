# ncu --set full of the fused disk front kernel (one config-5 step, FFT theta)
THETA=fft python tools/profile_step.py > gpurun_out/plain_fused.log 2>&1 && \
THETA=fft ncu --set full --clock-control none --import-source on -k regex:"disk_ftheta" -s 1 -c 1 \
   -o gpurun_out/prof_fused python tools/profile_step.py > gpurun_out/ncu_fused.log 2>&1; echo "ncu rc=$?"
