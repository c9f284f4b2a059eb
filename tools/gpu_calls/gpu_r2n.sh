#!/bin/bash
# round 2, call N: full validation + bench + reference arm + configs
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --durations=10 > gpurun_out/r2n_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_pytest.log
timeout 600 python bench.py > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2n_bench_ref.json 2> gpurun_out/r2n_bench_ref.err
timeout 600 python tools/run_configs.py 0 2 2s 4 3d > gpurun_out/r2n_configs.jsonl 2> gpurun_out/r2n_configs.err
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2n_e2e_timeline.txt 2>&1
