#!/bin/bash
# usage: tools/prof_round.sh TAG  -- ncu captures of the decode kernel per config + launch list
TAG=$1
export KVQ_SKIP_NVCC=1
for c in c2 c4 c3 c1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
     -o gpurun_out/prof_${c}_${TAG} python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${c}_${TAG}.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quant_append" --csv \
   --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
