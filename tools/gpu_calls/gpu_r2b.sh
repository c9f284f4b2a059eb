#!/bin/bash
# round 2, call B: changed kernels (cluster alias, lattice-shared B-spline sampler,
# chunked ties, sliced sharded merge, grouped Bluestein) -> tests, bench, configs, ncu
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
rc=$?; echo "smoke rc=$rc" >> gpurun_out/r2b_smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests/test_gpu_parity_ext.py tests/test_gpu_sharded.py tests/test_harness.py -m gpu -q -x --timeout 600 \
  --durations=10 > gpurun_out/r2b_pytest_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest_new.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_capi.py -m gpu -q -x --timeout 600 > gpurun_out/r2b_pytest_old.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_pytest_old.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?" >> gpurun_out/r2b_bench.err
timeout 600 python tools/run_configs.py 0 2 4 3d > gpurun_out/r2b_configs.jsonl 2> gpurun_out/r2b_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_step.csv \
  python tools/profile_step.py --warmup 2 --steps 2 > gpurun_out/r2b_ncu_step.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_cfg4.csv \
  python tools/run_config4_once.py > gpurun_out/r2b_ncu_cfg4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_cfg3.csv \
  python tools/run_config3_once.py > gpurun_out/r2b_ncu_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"alias_cluster|alias_planes|bluestein|fft_|gather_kernel|sample_poly_tcp" \
  -c 12 -o gpurun_out/r2b_step_full python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2b_ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sample_bspline_lat" \
  --launch-skip 7 -c 2 -o gpurun_out/r2b_cfg4_full python tools/run_config4_once.py > gpurun_out/r2b_ncu_cfg4_full.log 2>&1
ls -la gpurun_out >> gpurun_out/r2b_ncu_full.log
