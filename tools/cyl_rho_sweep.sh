mkdir -p gpurun_out
for c in 12 2 9 10 13 0 1 4; do
  export CURVIGPU_TILE_CFG="17,12,$c"
  CONFIGS=3 THETAS=fft timeout 120 python tools/kernel_times.py > gpurun_out/kt_cyl.jsonl 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/kt_cyl.jsonl').read().splitlines()[-1]);print('$c', [k['us'] for k in d['kernels']])"
done
