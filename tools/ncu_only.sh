export KVQ_SKIP_NVCC=1
O=gpurun_out
TAG=r1k
for c in c2 c4 c3 c1; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -f \
     -o $O/prof_${c}_$TAG python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_${c}_$TAG.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quant_append_kernel -s 2 -c 1 -f \
   -o $O/prof_k1c5_$TAG python tools/k1_bench.py int8 > $O/ncu_k1c5_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|quant_append" --csv \
   --log-file $O/launches_c2_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
