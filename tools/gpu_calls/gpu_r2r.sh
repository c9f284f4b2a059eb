#!/bin/bash
# round 2, call R: baseline of the restored tree (smoke, gpu tests, bench, step launch list)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2r_smoke.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x > gpurun_out/r2r_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2r_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2r_step_launches.csv python tools/profile_step.py > gpurun_out/r2r_ncu.log 2>&1
