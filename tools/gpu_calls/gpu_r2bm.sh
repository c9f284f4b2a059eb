#!/bin/bash
# round 2, call BM: counter-based alias kernels (A/B vs bitmaps), GPU suite, bench
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/alias_ab.py > gpurun_out/r2bm_alias_ab.jsonl 2>&1
SFFT_B200_ALIAS_COUNTERS=0 timeout 300 python tools/alias_ab.py >> gpurun_out/r2bm_alias_ab.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2bm_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bm_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2bm_bench.json 2> gpurun_out/r2bm_bench.err
