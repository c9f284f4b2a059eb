#!/bin/bash
# round 2, call E: alias A/B (cluster vs L2), config-2 host timeline and idle gaps, bench
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1 || exit 1
timeout 300 python tools/alias_ab.py > gpurun_out/r2e_alias_ab.jsonl 2>&1
SFFT_B200_ALIAS_CLUSTER=0 timeout 300 python tools/alias_ab.py >> gpurun_out/r2e_alias_ab.jsonl 2>&1
timeout 300 python tools/engine_gaps.py 2 > gpurun_out/r2e_gaps_cfg2.txt 2>&1
timeout 300 python tools/engine_timeline.py 2 > gpurun_out/r2e_timeline_cfg2.txt 2>&1
timeout 300 python tools/engine_gaps.py 4 > gpurun_out/r2e_gaps_cfg4.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_ext.py -m gpu -q -x --timeout 600 > gpurun_out/r2e_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_pytest.log
