mkdir -p gpurun_out
for c in default 17; do
  if [ $c = 17 ]; then export CURVIGPU_TILE_CFG=17; fi
  CONFIGS=5 THETAS=fft timeout 200 python tools/kernel_times.py > gpurun_out/kt_st$c.jsonl 2>&1; echo cfg $c; tail -1 gpurun_out/kt_st$c.jsonl
done
