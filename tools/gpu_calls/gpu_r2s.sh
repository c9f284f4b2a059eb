#!/bin/bash
# round 2, call S: ncu --set full of the three K2 kernels of a config-1 step
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2s_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_(colx2|row2048)_kernel" -s 5 -c 3 \
  -o gpurun_out/r2s_k2 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2s_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_ncu.log
