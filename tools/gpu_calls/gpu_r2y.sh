#!/bin/bash
# round 2, call Y: per-entry-point host time of the library calls
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/host_sections.py > gpurun_out/r2y_host_sections.txt 2>&1
