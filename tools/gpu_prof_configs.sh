# ncu --set full of one step of BASELINE configs 2, 3, 4 (fft theta where it applies)
python -m paper_2604_11558_b200.build > /dev/null
for k in 2 3 4; do
  CONFIG=$k THETA=fft python tools/profile_step.py > gpurun_out/plain_c$k.log 2>&1 && \
  CONFIG=$k THETA=fft timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|theta_|fbuild|disk_ftheta" -s 6 -c 8 \
     -o gpurun_out/prof_c$k python tools/profile_step.py > gpurun_out/ncu_c$k.log 2>&1; echo "ncu c$k rc=$?"; cat gpurun_out/plain_c$k.log | tail -1
done
