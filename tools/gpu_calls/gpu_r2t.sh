#!/bin/bash
# round 2, call T: speculative sampling start (presample) — tests, bench, e2e timeline
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_presample.py -q --timeout 300 -x > gpurun_out/r2t_presample.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_presample.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r2t_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2t_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2t_e2e_timeline.txt 2>&1
