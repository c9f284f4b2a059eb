#!/bin/bash
# round 2, call CI: measurement set of the restored final code (smoke, GPU suite, bench, configs incl. 3,
# bench launch list, reference arm)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ci_smoke.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2ci_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ci_pytest.log
timeout 900 python bench.py > gpurun_out/r2ci_bench.json 2> gpurun_out/r2ci_bench.err
timeout 1200 python tools/run_configs.py 0 2 2s 4 3d > gpurun_out/r2ci_configs.jsonl 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2ci_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2ci_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2ci_ncu.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2ci_reference.json 2> gpurun_out/r2ci_reference.err
