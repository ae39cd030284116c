#!/bin/bash
cd "$(dirname "$0")"
mkdir -p ../../gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > ../../gpurun_out/mb_clocks.csv &
SMI=$!
./fp64_peak > ../../gpurun_out/fp64_peak.json 2>&1
python blas_peak.py > ../../gpurun_out/blas_peak.json 2>&1
kill $SMI
nproc > ../../gpurun_out/host_cpu.txt; lscpu >> ../../gpurun_out/host_cpu.txt
cat ../../gpurun_out/fp64_peak.json ../../gpurun_out/blas_peak.json
