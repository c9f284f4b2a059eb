#!/bin/bash
# round 2, call AG: row upload on the copy stream overlapping the step preparation (e2e)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2ag_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ag_pytest.log
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2ag_e2e_timeline.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2ag_bench.json 2> gpurun_out/r2ag_bench.err
