# one config-5 step (fft theta): ncu --set full with source correlation of the front and the rho GEMM
mkdir -p gpurun_out
THETA=fft python tools/profile_step.py > gpurun_out/plain_step.log 2>&1; echo "plain rc=$?"
THETA=fft timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|disk_ftheta" -s 2 -c 2 \
   -o gpurun_out/prof_src ${NCU_EXTRA} python tools/profile_step.py > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
