for c in "2,0,0,0,0" "0,2,0,0,0" "0,0,2,0,0" "0,0,0,2,0" "0,0,0,0,2" "6,6,6,6,6" "1,1,1,1,1"; do
  CURVIGPU_TILE_CFG=$c DIMS="(100,96,100)" python tools/determinism2.py | sed "s/^/cfg $c: /"
done
