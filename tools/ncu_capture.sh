#!/bin/bash
# usage: tools/ncu_capture.sh TAG   -- ncu --set full of one K2 per config (C1-C5) of the in-tree
# build, written into gpurun_out/ncu_traffic_TAG.json tagged with the source hash (then copy it to
# profiles/ncu_traffic.json), plus the summaries.
TAG=${1:-cap}
export KVQ_SKIP_NVCC=1
O=gpurun_out
ARGS=""
for c in c2 c4 c3 c1 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -f \
     -o $O/prof_${c}_$TAG python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_${c}_$TAG.log 2>&1
  ARGS="$ARGS $c=$O/prof_${c}_$TAG.ncu-rep"
done
cp profiles/ncu_traffic.json $O/ncu_traffic_$TAG.json
python tools/ncu_traffic.py $O/ncu_traffic_$TAG.json $ARGS > $O/ncu_traffic_$TAG.log 2>&1
python tools/ncu_summary.py $O/prof_*_$TAG.ncu-rep > $O/ncu_summary_$TAG.txt 2>&1
