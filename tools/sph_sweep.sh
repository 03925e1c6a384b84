mkdir -p gpurun_out
for c in 12 13 11 7 9 2 17; do
  export CURVIGPU_TILE_CFG="$c"
  CONFIGS=2 THETAS=fft timeout 120 python tools/kernel_times.py > gpurun_out/kt_sph.jsonl 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/kt_sph.jsonl').read().splitlines()[-1]);print('$c', [k['us'] for k in d['kernels']])"
done
