#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity_ext.py tests/test_gpu_parity.py tests/test_gpu_guards.py -m gpu -q -x --timeout 600 > gpurun_out/r2g_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_pytest.log
timeout 600 python tools/run_configs.py 4 2 > gpurun_out/r2g_configs.jsonl 2> gpurun_out/r2g_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g_launches_cfg4.csv \
  python tools/run_config4_once.py > gpurun_out/r2g_ncu_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sample_bspline_chain" \
  --launch-skip 7 -c 1 -o gpurun_out/r2g_cfg4_full python tools/run_config4_once.py > gpurun_out/r2g_ncu_cfg4_full.log 2>&1
