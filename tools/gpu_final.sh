# round-end evidence: default bench line (extras), reference arm, launch list, ncu --set full of one
# config-5 step (fft + gemm) and of configs 2-4; summaries are written on the box (tools/ncu_summary.py)
# and the large .ncu-rep files dropped so gpurun_out stays under the 64 MiB copy-back limit
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench (defaults) rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench reference rc=$?"
SMALL="python bench.py --steps 1 --warmup 3 --chunk 20 --no-extras"
$SMALL > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py --launches gpurun_out/launches.csv > gpurun_out/launches_summary.txt
for t in fft gemm; do
  n=$([ $t = fft ] && echo 2 || echo 4)
  THETA=$t python tools/profile_step.py > gpurun_out/plain_step_$t.log 2>&1 && \
  THETA=$t timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64|resident_gemm|theta_|fbuild|disk_ftheta" -s $n -c $n \
     -o gpurun_out/prof_step_$t python tools/profile_step.py > gpurun_out/ncu_step_$t.log 2>&1; echo "ncu $t rc=$?"
done
python tools/ncu_summary.py gpurun_out/prof_step_fft.ncu-rep gpurun_out/prof_step_gemm.ncu-rep > gpurun_out/ncu_step_summary.txt
for k in 2 3 4; do
  CONFIG=$k THETA=fft python tools/profile_step.py > gpurun_out/plain_c$k.log 2>&1
  n=$(python -c "import json;print(len(json.load(open('gpurun_out/step_kernels_fft_c$k.json'))))")
  CONFIG=$k THETA=fft timeout 900 ncu --set full --clock-control none -k regex:"gemm_f64|resident_gemm|theta_|fbuild|disk_ftheta" -s $n -c $n \
     -o gpurun_out/prof_c$k python tools/profile_step.py > gpurun_out/ncu_c$k.log 2>&1; echo "ncu c$k rc=$?"
done
python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep gpurun_out/prof_c3.ncu-rep gpurun_out/prof_c4.ncu-rep > gpurun_out/ncu_c234_summary.txt
rm -f gpurun_out/prof_c*.ncu-rep gpurun_out/prof_step_gemm.ncu-rep
CONFIGS=5,1,2,3,4 THETAS=fft,gemm python tools/kernel_times.py > gpurun_out/kernel_times.jsonl 2>&1
python tools/step_times.py > gpurun_out/step_times.json 2>&1
du -sh gpurun_out; ls gpurun_out
head -c 1200 gpurun_out/bench_full.json; echo; cat gpurun_out/bench_ref.json
