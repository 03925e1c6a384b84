# one ncu --set full capture per kernel of one config-5 step, both theta modes
for t in fft gemm; do
  THETA=$t python tools/profile_step.py > gpurun_out/plain_step_$t.log 2>&1 && \
  THETA=$t ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|theta_|fbuild" -s 4 -c 8 \
     -o gpurun_out/prof_step_$t python tools/profile_step.py > gpurun_out/ncu_step_$t.log 2>&1; echo "ncu $t rc=$?"
done
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
