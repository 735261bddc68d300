#!/bin/bash
# A/B of kernel builds under sustained load: for each lib dir given, run
# tools/kbench.py --sustain S with that lib while nvidia-smi samples power and
# SM clock.  Output: gpurun_out/variant_<lib>.{json,csv}
S=${S:-8}
mkdir -p gpurun_out
for L in "$@"; do
  nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm,clocks_event_reasons.active -lms 250 --format=csv,noheader > gpurun_out/variant_$L.csv &
  SMI=$!
  COADAPT_LIB_PATH=$PWD/paper_2604_26687_b200/$L/libcoadapt_b200.so timeout 300 python tools/kbench.py --sustain $S --fused-gb 32 > gpurun_out/variant_$L.json 2>&1
  kill $SMI
  echo "$L $(cat gpurun_out/variant_$L.json | tail -1)"
done
