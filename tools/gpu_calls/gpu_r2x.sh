#!/bin/bash
# round 2, call X: host-time breakdown of the config-1 step and the e2e call; cProfiles
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/host_sections.py > gpurun_out/r2x_host_sections.txt 2>&1
timeout 300 python tools/api_cprofile.py > gpurun_out/r2x_api_cprofile.txt 2>&1
timeout 300 python tools/engine_gaps.py > gpurun_out/r2x_engine_gaps.txt 2>&1
timeout 300 python tools/engine_cprofile.py > gpurun_out/r2x_engine_cprofile.txt 2>&1
