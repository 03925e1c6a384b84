echo "--- baseline"; for i in 1 2; do CURVIGPU_TILE_CFG=0,0,2,0,0 REPS=12 python tools/chain_dbg.py | grep "stage 2 "; done
echo "--- direct epilogue"; for i in 1 2 3; do CURVIGPU_DIRECT_EPI=1 CURVIGPU_TILE_CFG=0,0,2,0,0 REPS=12 python tools/chain_dbg.py | grep "stage 2 "; done
