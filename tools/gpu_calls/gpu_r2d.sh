#!/bin/bash
# round 2, call D: alias cluster v3 (local full histograms + DSMEM fold),
# balanced B-spline chains
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/r2d_smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --durations=12 > gpurun_out/r2d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo "bench rc=$?" >> gpurun_out/r2d_bench.err
timeout 600 python tools/run_configs.py 0 2 4 3d > gpurun_out/r2d_configs.jsonl 2> gpurun_out/r2d_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_step.csv \
  python tools/profile_step.py --warmup 2 --steps 2 > gpurun_out/r2d_ncu_step.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches_cfg4.csv \
  python tools/run_config4_once.py > gpurun_out/r2d_ncu_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"alias_cluster|alias_planes" \
  -c 4 -o gpurun_out/r2d_alias_full python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2d_ncu_alias.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sample_bspline_chain" \
  --launch-skip 7 -c 2 -o gpurun_out/r2d_cfg4_full python tools/run_config4_once.py > gpurun_out/r2d_ncu_cfg4_full.log 2>&1
