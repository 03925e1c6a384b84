# build diagnostic variants of libcurvigpu.so (select with CURVIGPU_LIB=...)
cd /root/repo
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -shared -Iinclude"
S="paper_2604_11558_b200/csrc/plan.cu paper_2604_11558_b200/csrc/rng.cpp"
nvcc $F -DCG_REL_FENCE -o paper_2604_11558_b200/variants/vf.so $S &
nvcc $F -DCG_REL_DELAY -o paper_2604_11558_b200/variants/vb.so $S &
nvcc $F -o paper_2604_11558_b200/variants/vd.so $S &
wait
