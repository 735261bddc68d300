#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the single-GPU smoke
# (every kernel path incl. K1f M=16 shape 5 and the batched K1 ring) and, on
# 2 GPUs, over the NVLink slot exchange (standalone and in-pass).
# Output: gpurun_out/sanitize_*.txt and a summary line per run.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  CUDA_VISIBLE_DEVICES=0 timeout 900 $CS --tool $tool --error-exitcode 9 \
    python tools/sanitize_smoke.py > gpurun_out/sanitize_smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize smoke' gpurun_out/sanitize_smoke_$tool.txt | tr '\n' ' ')"
done
if [ "$(nvidia-smi -L | wc -l)" -ge 2 ]; then
  for tool in memcheck synccheck; do
    timeout 900 $CS --tool $tool --target-processes all --error-exitcode 9 \
      python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29610 tools/sanitize_p2p.py > gpurun_out/sanitize_p2p_$tool.txt 2>&1
    echo "p2p $tool rc=$? $(grep -E 'ERROR SUMMARY|sanitize p2p' gpurun_out/sanitize_p2p_$tool.txt | tr '\n' ' ')"
  done
fi
