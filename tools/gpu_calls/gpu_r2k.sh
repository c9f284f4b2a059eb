#!/bin/bash
# round 2, call K: batched gather loads
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_ext.py -m gpu -q -x --timeout 600 > gpurun_out/r2k_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2k_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
timeout 600 python tools/run_configs.py 2 4 > gpurun_out/r2k_configs.jsonl 2> gpurun_out/r2k_configs.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gather_kernel" \
  --launch-skip 0 -c 2 -o gpurun_out/r2k_fft_full python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2k_ncu_full.log 2>&1
