python -m paper_2604_11558_b200.build > /dev/null
python tools/coresidence_probe.py
CURVIGPU_GEMM_CPS=1 CURVIGPU_FRONT_CPS=1 python tools/coresidence_probe.py
CURVIGPU_GEMM_CPS=1 python tools/coresidence_probe.py
