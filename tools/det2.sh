python tools/determinism2.py
EAGER=1 python tools/determinism2.py
EAGER=1 SYNC=1 python tools/determinism2.py
CUDA_LAUNCH_BLOCKING=1 python tools/determinism2.py
DIMS="(10,12,10)" python tools/determinism2.py
DIMS="(100,100,100)" CURVIGPU_TILE_CFG=0 python tools/determinism2.py
DIMS="(96,100,96)" python tools/determinism2.py
DIMS="(100,96,100)" python tools/determinism2.py
