#!/bin/bash
# One ncu --set full capture of the dominant kernel of each BASELINE config,
# as bench.py launches it (after the warm-up), for roofline.traffic:
# /tmp/ncu_<cfg>.ncu-rep (stays on the box) + gpurun_out/ncu_<cfg>_{raw,details}.csv
mkdir -p gpurun_out
declare -A SKIPS=([c1]=4 [c2]=16 [c3]=16 [c4]=8)  # fused_tma launches per step
for cfg in ${CONFIGS:-c1 c2 c3 c4}; do
  SKIP=${SKIPS[$cfg]}
  CUDA_VISIBLE_DEVICES=0 timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:fused_tma_kernel --launch-skip $SKIP -c 1 -f -o /tmp/ncu_$cfg \
    python bench.py --config $cfg --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_${cfg}.log 2>&1
  ncu -i /tmp/ncu_$cfg.ncu-rep --page raw --csv > gpurun_out/ncu_${cfg}_raw.csv 2>/dev/null; ncu -i /tmp/ncu_$cfg.ncu-rep --page details --csv > gpurun_out/ncu_${cfg}_details.csv 2>/dev/null
  echo "$cfg rc=$? $(ls -la /tmp/ncu_$cfg.ncu-rep 2>/dev/null | awk '{print $5}')"
done
