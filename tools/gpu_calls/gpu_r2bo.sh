#!/bin/bash
# round 2, call BO: ncu --set full of the B-spline chain sampler (K1b) at config 4
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/run_config4_once.py > gpurun_out/r2bo_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bspline_chain --launch-skip 6 --launch-count 1 \
  -o gpurun_out/r2bo_k1b python tools/run_config4_once.py > gpurun_out/r2bo_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2bo_ncu.log
