# clipped bulk tensor stores for partial GEMM tiles (CURVIGPU_TMA_PARTIAL=1), re-tested with the proxy fence in place:
# bitwise rerun statistics on the n = 100 stages (ball, both theta modes), parity tests, kernel times
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
export CURVIGPU_LIB=$PWD/paper_2604_11558_b200/${LIB:-libcurvigpu.so}
O=gpurun_out/r02_tma_partial.txt; : > $O
for e in "" "CURVIGPU_TMA_PARTIAL=1" "CURVIGPU_TILE_CFG=19" "CURVIGPU_TMA_PARTIAL=1 CURVIGPU_TILE_CFG=19"; do
  for rep in 1 2; do echo "== kernel times [$e]" >> $O; env $e CONFIGS=4,3 timeout 300 python tools/kernel_times.py 2>&1 | cut -c1-330 >> $O; done
done
echo "== rerun statistics, CURVIGPU_TMA_PARTIAL=1" >> $O
CURVIGPU_TMA_PARTIAL=1 RS_CFGS=default,2,9,12,18,19 RS_CONFIGS=4,3 timeout 1500 python tools/race_stress.py ${REPS:-200} >> $O 2>&1
echo "== parity tests, CURVIGPU_TMA_PARTIAL=1" >> $O
CURVIGPU_TMA_PARTIAL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tensor.py tests/test_gpu_bulk_surface.py -x -q 2>&1 | tail -3 >> $O
python - <<'PY'
import json
for l in open('gpurun_out/r02_tma_partial.txt'):
    l=l.strip()
    if l.startswith('{"config"') and '"kernels"' in l:
        d=json.loads(l); print('c%d'%d['config'], [k['us'] for k in d['kernels']])
    elif l.startswith('{'):
        d=json.loads(l)
        if d.get('runs_differing'): print('DIFF', l)
    else: print(l[:200])
PY
grep -c runs_differing gpurun_out/r02_tma_partial.txt
