echo "--- baseline cfg2 stage 2"; for i in 1 2; do CURVIGPU_TILE_CFG=0,0,2,0,0 REPS=12 python tools/chain_dbg.py | grep "stage 2 "; done
echo "--- pad 40000 (1 CTA/SM)"; for i in 1 2; do CURVIGPU_SMEM_PAD=40000 CURVIGPU_TILE_CFG=0,0,2,0,0 REPS=12 python tools/chain_dbg.py | grep "stage 2 "; done
echo "--- non-persistent"; for i in 1 2; do CURVIGPU_NOPERSIST=1 CURVIGPU_TILE_CFG=0,0,2,0,0 REPS=12 python tools/chain_dbg.py | grep "stage 2 "; done
