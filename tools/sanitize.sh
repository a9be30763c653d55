#!/bin/bash
# compute-sanitizer over the small GPU cases: memcheck (out-of-bounds / misaligned
# accesses), racecheck (shared-memory hazards), synccheck (barrier misuse).
export KVQ_SKIP_NVCC=1
O=${1:-gpurun_out}
SEL="tests/test_gpu_quant.py tests/test_gpu_attention.py tests/test_gpu_session.py tests/test_gpu_prefix_transfer.py tests/test_gpu_sweep.py"
K="not fullsize and not race_free"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all \
     python -m pytest $SEL -q -x -k "$K" > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
done
