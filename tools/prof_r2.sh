#!/bin/bash
# usage: tools/prof_r2.sh TAG [configs...]
# Round-2 evidence in one GPU call, all under gpurun_out/:
#   bench_<cfg>_TAG.json     bench lines (K2 timed by its own grid span inside the PDL step)
#   prof_<cfg>_TAG.ncu-rep   ncu --set full of one K2 per config (same build)
#   ncu_traffic_TAG.json     dram bytes per launch of those captures, tagged with the source hash
#   launches_c2_TAG.csv      ncu launch list (gpu__time_duration) of a short default bench
TAG=${1:-r2}
shift
CFGS=${@:-c2 c3 c4 c1}
export KVQ_SKIP_NVCC=1
O=gpurun_out
for c in $CFGS; do
  timeout 400 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_${c}_$TAG.json 2> $O/bench_${c}_$TAG.err
done
cp profiles/ncu_traffic.json $O/ncu_traffic_$TAG.json 2>/dev/null
ARGS=""
for c in $CFGS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -f \
     -o $O/prof_${c}_$TAG python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_${c}_$TAG.log 2>&1
  ARGS="$ARGS $c=$O/prof_${c}_$TAG.ncu-rep"
done
python tools/ncu_traffic.py $O/ncu_traffic_$TAG.json $ARGS > $O/ncu_traffic_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quant_append" --csv \
   --log-file $O/launches_c2_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
