# measurement sweep: env settings x config-5 kernel times (EXPS="a=1 b=2;c=3")
mkdir -p gpurun_out
python -m paper_2604_11558_b200.build > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
IFS=';' read -ra LIST <<< "${EXPS}"
for e in "${LIST[@]}"; do
  echo "== $e"; env $e CONFIGS=${CONFIGS:-5} THETAS=${THETAS:-fft} timeout 300 python tools/kernel_times.py 2>&1 | tail -5 | cut -c1-400
done
