#!/bin/bash
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:fused_tma_kernel --launch-skip 8 -c 1 -f -o /tmp/ncu_c4src \
  python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_c4src.log 2>&1
ncu -i /tmp/ncu_c4src.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_c4_source_sass.csv 2>gpurun_out/ncu_c4src_err.txt
ls -la gpurun_out/ncu_c4_source_sass.csv
gzip -f gpurun_out/ncu_c4_source_sass.csv
