#!/bin/bash
# round 2, call CK: cProfile of a cold and a warm config-3 run
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/cfg3_cprofile.py > gpurun_out/r2ck_cfg3_cprofile.txt 2>&1
