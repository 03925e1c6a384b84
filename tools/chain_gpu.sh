mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "chained or ball" > gpurun_out/chain_tests.log 2>&1; echo "chain tests rc=$?"; tail -2 gpurun_out/chain_tests.log
CONFIGS=4 THETAS=fft timeout 120 python tools/kernel_times.py > gpurun_out/kt_chain.jsonl 2>&1; tail -2 gpurun_out/kt_chain.jsonl
CONFIG=4 THETA=fft timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64" -s 2 -c 1 \
   -o gpurun_out/prof_c4_chain python tools/profile_step.py > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
python tools/ncu_summary.py gpurun_out/prof_c4_chain.ncu-rep > gpurun_out/ncu_c4_chain_summary.txt; cat gpurun_out/ncu_c4_chain_summary.txt
