#!/bin/bash
# round 2, call DA (re-entry): full GPU suite, smoke, bench (both arms), configs, bench launch list
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02da_gpu_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02da_gpu_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02da_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r02da_bench.json 2> gpurun_out/r02da_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02da_bench_reference_arm.json 2> gpurun_out/r02da_bench_ref.err
timeout 900 python tools/run_configs.py > gpurun_out/r02da_configs.jsonl 2> gpurun_out/r02da_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02da_bench_launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/r02da_ncu.log 2>&1
tail -3 gpurun_out/r02da_gpu_pytest.txt; cat gpurun_out/r02da_smoke.txt | tail -2; cat gpurun_out/r02da_bench.json
