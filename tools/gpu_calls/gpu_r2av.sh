#!/bin/bash
# round 2, call AV: config-2 launch list (kernel times and grid sizes)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/run_config2_once.py > gpurun_out/r2av_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
  --log-file gpurun_out/r2av_cfg2_launches.csv python tools/run_config2_once.py > gpurun_out/r2av_ncu.log 2>&1
