# v9 evidence: full bench line, launch list, ncu --set full of one config-5 step (both theta modes)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
SMALL="python bench.py --steps 1 --warmup 3 --chunk 20 --no-extras"
$SMALL > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for t in fft gemm; do
  THETA=$t python tools/profile_step.py > gpurun_out/plain_step_$t.log 2>&1 && \
  THETA=$t timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|theta_|fbuild|disk_ftheta" -s $([ $t = fft ] && echo 2 || echo 4) -c 8 \
     -o gpurun_out/prof_step_$t python tools/profile_step.py > gpurun_out/ncu_step_$t.log 2>&1; echo "ncu $t rc=$?"
done
ls -la gpurun_out
