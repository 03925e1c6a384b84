# bench + ncu evidence (launch list, one --set full capture of the top GEMM)
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 2 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
SMALL="python bench.py --steps 1 --warmup 1 --chunk 20 --no-extras"
$SMALL > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
$SMALL > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -s 8 -c 3 -o gpurun_out/prof_gemm $SMALL > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
$SMALL > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fbuild -s 2 -c 1 -o gpurun_out/prof_fbuild $SMALL > gpurun_out/ncu_full_fb.log 2>&1; echo "ncu fbuild rc=$?"
ls -la gpurun_out
