#!/bin/bash
# round 2, call AH: odd row stride for the mixed-radix column tiles (bank conflicts)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python tools/k2_ab.py > gpurun_out/r2ah_k2.jsonl 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r2ah_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/r2ah_pytest.log
timeout 300 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2ah_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r2ah_step_launches.csv python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r2ah_ncu.log 2>&1
