#!/bin/bash
# round 2, call U: step-level K split + speculative sampling; pipelined Bluestein groups (A/B)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_presample.py -q --timeout 300 > gpurun_out/r2u_presample.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_presample.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2u_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2u_bench.json 2> gpurun_out/r2u_bench.err
for mb in 0 8 32; do
SFFT_B200_FFT_PIPE_MB=$mb timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2u_bench_pipe$mb.json 2> gpurun_out/r2u_bench_pipe$mb.err
done
timeout 300 python tools/e2e_timeline.py > gpurun_out/r2u_e2e_timeline.txt 2>&1
timeout 300 python tools/bench_timeline.py > gpurun_out/r2u_bench_timeline.txt 2>&1
