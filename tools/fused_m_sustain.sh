#!/bin/bash
mkdir -p gpurun_out
for R in 1 2; do for M in 16 8 4; do
  nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm --format=csv,noheader -lms 250 > gpurun_out/r02ff_m${M}_r$R.csv &
  SMI=$!
  timeout 300 python tools/kbench.py --sustain 6 --fused-gb 32 --fused-m $M --kernels k1f > gpurun_out/r02ff_m${M}_r$R.json 2>&1
  kill $SMI
  echo "M=$M r$R $(tail -1 gpurun_out/r02ff_m${M}_r$R.json) clk=$(awk -F', ' '{split($3,a," "); if ($2+0>850) print a[1]}' gpurun_out/r02ff_m${M}_r$R.csv | sort -n | awk '{v[NR]=$1} END {print v[int(NR/2)+1]}')"
done; done
