python -m paper_2604_11558_b200.build > /dev/null
for c in 1 4 8; do
  BENCH_E2E_CHUNKS=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-extras --theta fft > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_c$c.json'))
print('chunks $c value %.4e'%d['value'], 'e2e %.4e'%d['e2e']['value'], 'ratio', round(d['e2e']['value']/d['value'],4))"
done
timeout 1200 python -m pytest tests -x -q -m gpu -k "ensemble or Ensemble" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
