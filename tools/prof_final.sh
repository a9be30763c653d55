#!/bin/bash
# usage: tools/prof_final.sh TAG
# End-of-round evidence from one build, all under gpurun_out/:
#   gputests_TAG.txt          pytest -m gpu + smoke()
#   bench_<cfg>_TAG.json      bench lines: default (C2 + cpu_baseline), reference arm, c1..c5, c5 fp8,
#                             --serving (32 layers), widened rows (multi-query, transfer, host tier)
#   prof_<cfg>_TAG.ncu-rep    ncu --set full of one K2 per config and of K1 at the C5 step shape
#                             (summarised into ncu_summary_TAG.txt; only C4's and K1's reports are kept)
#   ncu_traffic_TAG.json      dram bytes per launch of those captures, tagged with the source hash
#   launches_c2_TAG.csv       ncu launch list (gpu__time_duration) of a short default bench
#   sass_TAG.txt              static SASS mix (tools/sass_mix.py, tools/sass_pageloop.py)
#   sanitize_*.log            compute-sanitizer memcheck / racecheck / synccheck
TAG=${1:-final}
export KVQ_SKIP_NVCC=1
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/gputests_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" >> $O/gputests_$TAG.txt 2>&1
timeout 400 python bench.py > $O/bench_default_$TAG.json 2> $O/bench_default_$TAG.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference_$TAG.json 2>&1
for c in c2 c1 c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_${c}_$TAG.json 2>>$O/bench_err_$TAG.txt
done
timeout 300 python bench.py --config c5 --kv fp8_e4m3 --steps 100 --warmup 5 --no-cpu-baseline > $O/bench_c5fp8_$TAG.json 2>>$O/bench_err_$TAG.txt
timeout 300 python bench.py --serving --layers 32 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_serving_$TAG.json 2>>$O/bench_err_$TAG.txt
timeout 300 python tools/bench_widened.py > $O/widened_$TAG.jsonl 2>>$O/bench_err_$TAG.txt
python tools/sass_mix.py "quant_append|decode_kernel" > $O/sass_$TAG.txt 2>&1
python tools/sass_pageloop.py >> $O/sass_$TAG.txt 2>&1
ARGS=""
for c in c2 c4 c3 c1 c5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -f \
     -o $O/prof_${c}_$TAG python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_${c}_$TAG.log 2>&1
  ARGS="$ARGS $c=$O/prof_${c}_$TAG.ncu-rep"
done
timeout 600 ncu --set full --metrics lts__t_sectors_op_write.sum --clock-control none --import-source on \
   -k regex:quant_append_tile -s 2 -c 1 -f -o $O/prof_k1c5_$TAG python tools/k1_bench.py int8 > $O/ncu_k1c5_$TAG.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic_$TAG.json
python tools/ncu_traffic.py $O/ncu_traffic_$TAG.json $ARGS > $O/ncu_traffic_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quant_append" --csv \
   --log-file $O/launches_c2_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_summary.py $O/prof_c2_$TAG.ncu-rep $O/prof_c4_$TAG.ncu-rep $O/prof_c3_$TAG.ncu-rep \
   $O/prof_c1_$TAG.ncu-rep $O/prof_c5_$TAG.ncu-rep $O/prof_k1c5_$TAG.ncu-rep > $O/ncu_summary_$TAG.txt 2>&1
# gpurun copies back <= 64 MiB: keep the summaries and C4's report (the source view of the g = 16 kernel)
rm -f $O/prof_c2_$TAG.ncu-rep $O/prof_c3_$TAG.ncu-rep $O/prof_c1_$TAG.ncu-rep $O/prof_c5_$TAG.ncu-rep
bash tools/sanitize.sh $O > $O/sanitize_$TAG.txt 2>&1
rm -f $O/sanitize_*.log.tmp
echo done
