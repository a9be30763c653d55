#!/bin/bash
# usage: tools/prof_one.sh TAG CONFIG
export KVQ_SKIP_NVCC=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
   -o gpurun_out/prof_$2_$1 python bench.py --config $2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$2_$1.log 2>&1
