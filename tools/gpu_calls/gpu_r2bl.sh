#!/bin/bash
# round 2, call BL: deferred stream spawns, device line points
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2bl_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bl_pytest.log
timeout 300 python tools/host_sections.py > gpurun_out/r2bl_host_sections.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2bl_bench.json 2> gpurun_out/r2bl_bench.err
timeout 1200 python tools/run_configs.py 0 2 2s 4 > gpurun_out/r2bl_configs.jsonl 2>&1
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2bl_e2e_timeline.txt 2>&1
