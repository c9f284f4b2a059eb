#!/bin/bash
# round 2, call AE: overlapped engine steps (settled counts), tests, configs, bench
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_engine_overlap.py -q --timeout 300 > gpurun_out/r2ae_overlap.log 2>&1
echo "rc=$?" >> gpurun_out/r2ae_overlap.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2ae_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ae_pytest.log
timeout 600 python tools/run_configs.py 0 2 2s 4 > gpurun_out/r2ae_configs.jsonl 2>&1
timeout 300 python tools/engine_gaps.py > gpurun_out/r2ae_engine_gaps.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2ae_bench.json 2> gpurun_out/r2ae_bench.err
