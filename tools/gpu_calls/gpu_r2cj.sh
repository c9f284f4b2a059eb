#!/bin/bash
# round 2, call CJ: bench-step timeline of the current code; config 3 twice in one process
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/bench_timeline.py > gpurun_out/r2cj_bench_timeline.txt 2>&1
timeout 600 python tools/cfg3_twice.py > gpurun_out/r2cj_cfg3_twice.txt 2>&1
