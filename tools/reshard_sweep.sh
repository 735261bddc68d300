#!/bin/bash
# KX (reshard pull/push) bandwidth on >= 2 GPUs: the timed TP->PP transition
# of tests/mp_reshard_worker.py (537 MB per rank), pull and push.  The tuning
# sweep that chose csrc/reshard.cu's constants is profiles/r01_reshard_sweep.txt.
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=${NPROC:-2} \
  --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tests/mp_reshard_worker.py \
  2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ok"], [[(t["mode"], round(t["wire_gbs"]), round(t["ms"],3)) for t in r] for r in d["bandwidth"]])'
