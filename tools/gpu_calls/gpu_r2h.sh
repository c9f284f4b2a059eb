#!/bin/bash
# round 2, call H: full validation + bench + configs + e2e timeline + launch lists
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 --durations=10 > gpurun_out/r2h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
echo "bench rc=$?" >> gpurun_out/r2h_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2h_bench_ref.json 2> gpurun_out/r2h_bench_ref.err
timeout 600 python tools/run_configs.py 0 2 2s 4 3d > gpurun_out/r2h_configs.jsonl 2> gpurun_out/r2h_configs.err
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2h_e2e_timeline.txt 2>&1
timeout 300 python tools/engine_gaps.py 2 > gpurun_out/r2h_gaps_cfg2.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2h_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_ncu_bench.log 2>&1
