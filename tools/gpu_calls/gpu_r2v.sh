#!/bin/bash
# round 2, call V: persistent pipelined Bluestein row pass (A/B vs one row per CTA)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/k2_ab.py > gpurun_out/r2v_k2_ab.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2v_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2v_pytest.log
