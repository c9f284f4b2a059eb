#!/bin/bash
# round 2, call AI: where config 4's wall goes (GPU gaps, host profile)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/engine_gaps.py 4 > gpurun_out/r2ai_engine_gaps_cfg4.txt 2>&1
timeout 300 python tools/engine_cprofile.py 4 > gpurun_out/r2ai_engine_cprofile_cfg4.txt 2>&1
