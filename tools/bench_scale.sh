#!/bin/bash
# Multi-GPU scaling of the default workload (C2) and the sharded configs, fused
# peer gather vs the NCCL all-gather baseline.  Needs N GPUs on one node.
#   tools/bench_scale.sh [configs] [gpu counts]
CFGS=${1:-"c2 c3 c4"}
NS=${2:-"1 2 4 8"}
export KVQ_SKIP_NVCC=1
for c in $CFGS; do
  for n in $NS; do
    for g in peer nccl; do
      if [ "$n" = 1 ]; then
        [ "$g" = nccl ] && continue
        timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline
      else
        timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port $((29500 + n)) bench.py --gpus $n --config $c --gather $g --steps 100 --warmup 5
      fi | tail -n 1 | python3 -c "
import json, sys
d = json.loads(sys.stdin.read())
print('$c', 'N=$n', '$g', 'tok/s %.0f' % d['value'], 'step_ms %.4f' % d['ms_per_step'],
      'e2e_ms %.4f' % d['e2e']['ms_per_step'], d['config'].get('parallelism'))"
    done
  done
done
