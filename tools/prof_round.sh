#!/bin/bash
# usage: tools/prof_round.sh TAG
# One GPU call's worth of round evidence, all under gpurun_out/:
#   bench_default_TAG.json   default bench line (C2, with cpu_baseline)
#   bench_reference_TAG.json --impl reference line
#   bench_all_TAG.txt        c2 c1 c3 c4 c5 (+ c5 fp8) summaries
#   prof_<cfg>_TAG.ncu-rep   ncu --set full of K2 per config, K1 at the C5 step shape
#   launches_c2_TAG.csv      ncu launch list (gpu__time_duration) of a short default bench
TAG=${1:-r}
export KVQ_SKIP_NVCC=1
O=gpurun_out
timeout 400 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_$TAG.json 2>&1
for c in c2 c1 c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_${c}_$TAG.json 2>&1
done
timeout 300 python bench.py --config c5 --kv fp8_e4m3 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_c5fp8_$TAG.json 2>&1
for c in c2 c4 c3 c1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -f \
     -o $O/prof_${c}_$TAG python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_${c}_$TAG.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_append_kernel -s 2 -c 1 -f \
   -o $O/prof_k1c5_$TAG python tools/k1_bench.py int8 > $O/ncu_k1c5_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quant_append" --csv \
   --log-file $O/launches_c2_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
