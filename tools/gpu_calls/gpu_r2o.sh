#!/bin/bash
# round 2, call O: chain sampler chirp prefetch + occupancy-sized grid; bench twice (cold-step variance)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity_ext.py tests/test_gpu_guards.py -m gpu -q --timeout 600 > gpurun_out/r2o_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_pytest.log
timeout 600 python tools/run_configs.py 4 > gpurun_out/r2o_configs.jsonl 2> gpurun_out/r2o_configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2o_launches_cfg4.csv \
  python tools/run_config4_once.py > gpurun_out/r2o_ncu_cfg4.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-d10 > gpurun_out/r2o_bench1.json 2> gpurun_out/r2o_bench1.err
timeout 600 python bench.py --no-cpu-baseline --no-d10 > gpurun_out/r2o_bench2.json 2> gpurun_out/r2o_bench2.err
