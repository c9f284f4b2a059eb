#!/bin/bash
# round 2, call AX: cold-cache d=10 walls with / without table building in the step preparation
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for rep in 1 2; do
SFFT_B200_PREP_TABLES=0 timeout 600 python tools/cold_ab.py >> gpurun_out/r2ax_cold_ab.jsonl 2>&1
SFFT_B200_PREP_TABLES=1 timeout 600 python tools/cold_ab.py >> gpurun_out/r2ax_cold_ab.jsonl 2>&1
done
