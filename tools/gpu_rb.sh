python tools/fbuild_time.py
for r in 2 8; do CURVIGPU_LIB=paper_2604_11558_b200/variants/rb$r.so python tools/fbuild_time.py; done
