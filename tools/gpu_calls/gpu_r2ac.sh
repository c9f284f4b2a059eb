#!/bin/bash
# round 2, call AD: next step enqueued during the current one (speculative count)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r2ac_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ac_pytest.log
timeout 600 python tools/run_configs.py 0 2 2s 4 > gpurun_out/r2ac_configs.jsonl 2>&1
timeout 300 python tools/engine_gaps.py > gpurun_out/r2ac_engine_gaps.txt 2>&1
