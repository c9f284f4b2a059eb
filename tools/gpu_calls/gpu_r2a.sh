#!/bin/bash
# round 2, call A: GPU tests (incl. the new extended parity), sanitizer passes, a short bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 600 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_step.py > gpurun_out/r2a_memcheck.log 2>&1
echo "memcheck rc=$?" >> gpurun_out/r2a_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_step.py 3000 > gpurun_out/r2a_racecheck.log 2>&1
echo "racecheck rc=$?" >> gpurun_out/r2a_racecheck.log
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_step.py 3000 > gpurun_out/r2a_synccheck.log 2>&1
echo "synccheck rc=$?" >> gpurun_out/r2a_synccheck.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench rc=$?" >> gpurun_out/r2a_bench.err
