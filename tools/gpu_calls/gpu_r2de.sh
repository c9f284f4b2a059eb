#!/bin/bash
# round 2, call DE: stability evidence of the final code (compute-sanitizer is closed on this pool): the GPU suite three
# times in a row, 10000 further fuzz seeds, the bench in three fresh processes
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
out=gpurun_out/r02de_stability.txt
: > $out
for i in 1 2 3; do
  timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -1 >> $out
done
echo "fuzz seeds 4000..13999:" >> $out
SFFT_B200_FUZZ_BASE=4000 SFFT_B200_FUZZ_CASES=10000 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q 2>&1 | tail -1 >> $out
for i in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bench process $i:', 'value', round(d['value']), 'ms_per_step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'K1 ms', round(d['kernels_ms']['sample_poly'],4), 'clocks', d['clocks'])" >> $out
done
cat $out
