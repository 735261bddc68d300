#!/bin/bash
# A/B/A/B of K1f launch shapes (COADAPT_TMA_SHAPE; needs a library built with
# make EXTRA_NVFLAGS=-DCOADAPT_SHAPE_SWEEP=1) on one box under sustained
# load, with power / SM clock sampling: gpurun_out/<TAG>_s<shape>_r<round>.*
S=${S:-6}; ROUNDS=${ROUNDS:-2}; TAG=${TAG:-shape}; M=${M:-16}
mkdir -p gpurun_out
for R in $(seq 1 $ROUNDS); do
  for V in "$@"; do
    out=gpurun_out/${TAG}_s${V}_r$R
    nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm,clocks_event_reasons.active -lms 250 --format=csv,noheader > $out.csv &
    SMI=$!
    COADAPT_TMA_SHAPE=$V timeout 300 python tools/kbench.py --sustain $S --fused-gb 32 --fused-m $M --kernels k1f > $out.json 2>&1
    kill $SMI
    echo "shape $V r$R $(tail -1 $out.json)"
  done
done
