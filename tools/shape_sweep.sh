#!/bin/bash
# fused_tma_kernel shape sweep: burst and sustained K1f GB/s per (M, shape).
# usage: [SUSTAIN=6] tools/shape_sweep.sh "16 8" "4 5 0"   -> gpurun_out/shape_sweep.txt
# (the library must be built with make EXTRA_NVFLAGS=-DCOADAPT_SHAPE_SWEEP=1;
#  the shipped build instantiates only the best shape per M)
out=gpurun_out/shape_sweep.txt; mkdir -p gpurun_out; : > $out
for M in $1; do for V in $2; do
  b=$(COADAPT_TMA_SHAPE=$V timeout 120 python tools/kbench.py --kernels k1f --fused-m $M --fused-gb 32 --reps 10 | tail -1)
  if [ -n "$SUSTAIN" ]; then
    s=$(COADAPT_TMA_SHAPE=$V timeout 120 python tools/kbench.py --kernels k1f --fused-m $M --fused-gb 32 --sustain $SUSTAIN | tail -1)
    s=$(echo $s | python -c 'import json,sys;print(json.load(sys.stdin)["k1f_gbs"])')
  else s=-; fi
  echo "M=$M shape=$V burst=$(echo $b | python -c 'import json,sys;print(json.load(sys.stdin)["k1f_gbs"])') sustained=$s" | tee -a $out
done; done
