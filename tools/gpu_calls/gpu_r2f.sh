#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/engine_cprofile.py --callees > gpurun_out/r2f_cprofile_cfg2.txt 2>&1
timeout 300 python tools/alias_ab.py > gpurun_out/r2f_alias_ab.jsonl 2>&1
