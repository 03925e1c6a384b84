#!/bin/bash
# FP64 peak probe with clocks sampled during the run
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peak_clocks.csv &
SMI=$!
./tools/fp64_peak > gpurun_out/fp64_peak.log 2>&1
kill $SMI
nvidia-smi > gpurun_out/nvidia_smi.txt
lscpu > gpurun_out/lscpu.txt
nproc >> gpurun_out/lscpu.txt
cat gpurun_out/fp64_peak.log
