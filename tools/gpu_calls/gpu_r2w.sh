#!/bin/bash
# round 2, call W: fused cooperative alias kernel (A/B, parity, full GPU suite, bench)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for v in fused l2; do
  if [ $v = l2 ]; then export SFFT_B200_ALIAS_FUSED=0; fi
  timeout 300 python tools/alias_ab.py >> gpurun_out/r2w_alias_ab.jsonl 2>&1
done
unset SFFT_B200_ALIAS_FUSED
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2w_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
