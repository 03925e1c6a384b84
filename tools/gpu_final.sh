# round-end evidence: full bench line (extras), launch list, ncu --set full of one config-5 step (fft + gemm)
mkdir -p gpurun_out
python -m paper_2604_11558_b200.build > /dev/null
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
SMALL="python bench.py --steps 1 --warmup 3 --chunk 20 --no-extras"
$SMALL > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for t in fft gemm; do
  THETA=$t python tools/profile_step.py > gpurun_out/plain_step_$t.log 2>&1 && \
  THETA=$t timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|theta_|fbuild|disk_ftheta" -s $([ $t = fft ] && echo 2 || echo 4) -c 8 \
     -o gpurun_out/prof_step_$t python tools/profile_step.py > gpurun_out/ncu_step_$t.log 2>&1; echo "ncu $t rc=$?"
done
for k in 2 3 4; do
  CONFIG=$k THETA=fft python tools/profile_step.py > gpurun_out/plain_c$k.log 2>&1
  n=$(python -c "import json;print(len(json.load(open('gpurun_out/step_kernels_fft_c$k.json'))))")
  CONFIG=$k THETA=fft timeout 900 ncu --set full --clock-control none -k regex:"gemm_f64|theta_|fbuild|disk_ftheta" -s $n -c $n \
     -o gpurun_out/prof_c$k python tools/profile_step.py > gpurun_out/ncu_c$k.log 2>&1; echo "ncu c$k rc=$?"
done
CONFIGS=1,2,3,4 THETAS=fft,gemm python tools/kernel_times.py > gpurun_out/kernel_times.jsonl 2>&1
python tools/step_times.py > gpurun_out/step_times.json 2>&1
ls gpurun_out
