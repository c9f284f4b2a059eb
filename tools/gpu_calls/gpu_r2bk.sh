#!/bin/bash
# round 2, call BK: host micro-optimizations (table-cache lookup, primes memo, library zero fill, get_device)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2bk_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bk_pytest.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-d10 > gpurun_out/r2bk_bench$i.json 2>/dev/null; done
timeout 600 python tools/gc_ab.py > gpurun_out/r2bk_cfg2_walls.jsonl 2>&1
