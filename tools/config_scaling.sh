#!/bin/bash
# bench.py lines for every BASELINE config at N = 1, 2, 4 (one box), e2e on,
# CPU baseline off; one JSON line per run into gpurun_out/scaling_<cfg>_n<N>.json
for c in ${CONFIGS:-c1 c2 c3 c4}; do for n in ${NS:-1 2 4}; do
  if [ "$n" = 1 ]; then
    timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu 2>/dev/null | grep '^{' | tail -1 > gpurun_out/scaling_${c}_n$n.json
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29800 + n)) bench.py --gpus $n --config $c --steps 10 --warmup 3 2>/dev/null \
      | grep '^{' | tail -1 > gpurun_out/scaling_${c}_n$n.json
  fi
  python -c "import json; d=json.load(open('gpurun_out/scaling_${c}_n$n.json')); print('$c', d['n_gpus'], d['value'], d['roofline']['frac'], d['e2e']['value'] if d['e2e'] else None, d['clocks']['sm_mhz'], d['goodput_step']['step_ms'])"
done; done
