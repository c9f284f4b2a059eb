#!/bin/bash
# round 2, call I: early step preparation in reconstruct_step (e2e), k1-outer Bluestein row order
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2i_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2i_e2e_timeline.txt 2>&1
timeout 600 python tools/run_configs.py 2 4 > gpurun_out/r2i_configs.jsonl 2> gpurun_out/r2i_configs.err
