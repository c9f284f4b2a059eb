#!/bin/bash
# round 2, call AL: ncu --set full of K1 (sample_poly_tcp_kernel) in a config-1 step
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2al_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sample_poly_tcp_kernel" -s 1 -c 1 \
  -o gpurun_out/r2al_k1 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2al_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2al_ncu.log
