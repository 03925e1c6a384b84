mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "chained or ball" > gpurun_out/chain_tests.log 2>&1; echo "chain tests rc=$?"; tail -2 gpurun_out/chain_tests.log
for c in 14 15; do CURVIGPU_CHAIN_CFG=$c CONFIGS=4 THETAS=fft timeout 120 python tools/kernel_times.py > gpurun_out/kt_chain$c.jsonl 2>&1; echo cfg $c; tail -1 gpurun_out/kt_chain$c.jsonl; done
