SMALL="python bench.py --steps 1 --warmup 1 --chunk 20 --no-extras"
export CURVIGPU_NO_FUSED_FRONT=1
$SMALL > gpurun_out/plain_t.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"theta_fast|fbuild_rows" -s 4 -c 2 -o gpurun_out/prof_theta $SMALL > gpurun_out/ncu_theta.log 2>&1; echo "ncu theta rc=$?"
unset CURVIGPU_NO_FUSED_FRONT
$SMALL > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"disk_ftheta" -s 2 -c 1 -o gpurun_out/prof_fused $SMALL > gpurun_out/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
