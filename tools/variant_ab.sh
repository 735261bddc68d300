#!/bin/bash
# A/B/A/B of kernel builds under sustained load on one box: for each round
# and each lib dir given, tools/kbench.py --sustain S (K1 8 GB bucket, K1f
# M=16 x 2 GB) while nvidia-smi samples power / SM clock every 250 ms.
# Output: gpurun_out/ab_<tag>_<lib>_r<round>.{json,csv}
S=${S:-6}
ROUNDS=${ROUNDS:-2}
TAG=${TAG:-ab}
KERNELS=${KERNELS:-k1,k1f}
mkdir -p gpurun_out
for R in $(seq 1 $ROUNDS); do
  for L in "$@"; do
    out=gpurun_out/${TAG}_${L}_r$R
    nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm,clocks_event_reasons.active -lms 250 --format=csv,noheader > $out.csv &
    SMI=$!
    COADAPT_LIB_PATH=$PWD/paper_2604_26687_b200/$L/libcoadapt_b200.so timeout 300 \
      python tools/kbench.py --sustain $S --fused-gb 32 --kernels $KERNELS > $out.json 2>&1
    kill $SMI
    echo "$L r$R $(tail -1 $out.json)"
  done
done
