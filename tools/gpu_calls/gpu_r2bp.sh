#!/bin/bash
# round 2, call BP: K1b at 3 CTAs per SM (launch bounds)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k "bspline or config4 or cfg4" > gpurun_out/r2bp_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2bp_pytest.log
timeout 300 python tools/run_config4_once.py > gpurun_out/r2bp_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bspline" --csv --log-file gpurun_out/r2bp_cfg4_bspline.csv python tools/run_config4_once.py > gpurun_out/r2bp_ncu.log 2>&1
