python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python tools/determinism.py 2>&1 | grep -c "deterministic=True"; python tools/determinism.py 2>&1 | grep "False"
for t in fft gemm; do
  python bench.py --steps 3 --warmup 2 --no-extras --theta $t > gpurun_out/bench_$t.json 2> gpurun_out/bench_$t.err; echo "bench $t rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$t.json'))
print('$t value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"
done
