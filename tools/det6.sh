for i in 1 2 3; do CURVIGPU_TILE_CFG=0,0,2,0,0 python tools/chain_dbg2.py | grep -E "rep|first bad"; echo run$i; done
for i in 1 2; do DIMS="(100,100,100)" python tools/determinism2.py; done
python tools/determinism.py 2>&1 | grep -v "deterministic=True"
echo determinism-done
