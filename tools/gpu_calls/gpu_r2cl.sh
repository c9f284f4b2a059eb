#!/bin/bash
# round 2, call CL: post-chirp recomputed in the inverse column pass: chirp test, K2 A/B (config 1),
# GPU suite, bench, configs 2/4, bench launch list
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_chirp.py -q -x > gpurun_out/r2cl_chirp_test.log 2>&1; echo rc=$? >> gpurun_out/r2cl_chirp_test.log
for i in 1 2; do timeout 600 python tools/k2_ab.py --reps 30 >> gpurun_out/r2cl_k2_ab.jsonl 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r2cl_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r2cl_pytest.log
for v in 1 0 1 0; do
  SFFT_B200_CHIRP_TABLE=$v timeout 600 python bench.py --no-cpu-baseline --no-d10 > gpurun_out/r2cl_b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2cl_b.json').read().strip().splitlines()[-1]); print('table=$v', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2), d['kernels_ms'])" >> gpurun_out/r2cl_bench_ab.txt
done
for v in 1 0; do SFFT_B200_CHIRP_TABLE=$v timeout 900 python tools/run_configs.py 2 4 > gpurun_out/r2cl_configs_table$v.jsonl 2>&1; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2cl_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2cl_bench_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2cl_ncu.log 2>&1
