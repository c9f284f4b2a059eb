# wide-J1 (small B panels) A/B: parity tests, bench both ways twice, timeline
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_ext.py tests/test_gpu_sharded.py -q -x --timeout 600 > gpurun_out/r2cg_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2cg_pytest.log
for v in 1 0 1 0; do
  SFFT_B200_J1_WIDE=$v timeout 600 python bench.py --no-cpu-baseline --no-d10 > gpurun_out/r2cg_b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/r2cg_b.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2), d['kernels_ms'], d['roofline']['traffic'])" >> gpurun_out/r2cg_ab.txt
done
SFFT_B200_J1_WIDE=1 python tools/bench_timeline.py > gpurun_out/r2cg_timeline_1.txt 2>&1
SFFT_B200_J1_WIDE=0 python tools/bench_timeline.py > gpurun_out/r2cg_timeline_0.txt 2>&1
