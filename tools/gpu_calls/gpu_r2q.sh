#!/bin/bash
# round 2, call Q: e2e without the extent read-back before the alias kernel
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q_smoke.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r2q_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2q_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2q_e2e_timeline.txt 2>&1
