mkdir -p gpurun_out
CONFIGS=3,4 THETAS=fft timeout 300 python tools/kernel_times.py > gpurun_out/kt_fb.jsonl 2>&1; cut -c1-120 gpurun_out/kt_fb.jsonl
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "apply_diffusion or full_config or small_config" 2>&1 | tail -1
