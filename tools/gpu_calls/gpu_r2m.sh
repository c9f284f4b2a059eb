#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q --timeout 600 > gpurun_out/r2m_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2m_pytest.log
