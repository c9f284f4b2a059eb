#!/bin/bash
# round 2, call DD: bench of the final code with the per-class DRAM traffic of the r02dc capture in its rooflines
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python bench.py > gpurun_out/r02dd_bench.json 2> gpurun_out/r02dd_bench.err; echo "rc=$?"
tail -c 600 gpurun_out/r02dd_bench.err
