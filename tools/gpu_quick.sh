# build, GPU tests, quick config-5 bench (fft), per-config
python -m paper_2604_11558_b200.build > /dev/null
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for t in ${THETAS:-fft}; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --theta $t > gpurun_out/bench_$t.json 2> gpurun_out/bench_$t.err; echo "bench $t rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_$t.json'))
print('$t value %.4e'%d['value'], 'ms/step', round(d['ms_per_step'],2))
for r in d['kernels']: print('  ', r['kernel'], round(r['achieved'],2), r['unit'], round(r['frac'],3), round(r['ms_per_launch'],4))
"
done
[ -n "$PERCONFIG" ] && timeout 600 python tools/per_config.py 2>&1 | tee gpurun_out/per_config.jsonl | cut -c1-100
true
