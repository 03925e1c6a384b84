# state check on one B200: GPU tests, smoke, bench in both theta modes, fused vs unfused front
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
for v in fft gemm; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --theta $v > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo "bench $v rc=$?"
done
CURVIGPU_NO_FUSED_FRONT=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --theta fft > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err; echo "bench unfused rc=$?"
for f in fft gemm unfused; do python -c "
import json; d=json.load(open('gpurun_out/bench_$f.json'))
print('$f value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2), 'e2e', d.get('e2e',{}).get('value'))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"; done
