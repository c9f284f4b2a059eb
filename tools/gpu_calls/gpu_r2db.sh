#!/bin/bash
# round 2, call DB: extended randomised parity (3000 further seeds), ncu --set full of the config-1 step kernels of the final code
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
SFFT_B200_FUZZ_BASE=1000 SFFT_B200_FUZZ_CASES=3000 timeout 1800 python -m pytest tests/test_gpu_fuzz.py -m gpu -q > gpurun_out/r02db_fuzz_extended.txt 2>&1
echo "rc=$?" >> gpurun_out/r02db_fuzz_extended.txt
timeout 300 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r02db_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"sample_poly_tcp|fft_colx|fft_row2048|gather_kernel|alias_c|poly_bpanel" --launch-skip 8 --launch-count 10 \
  -o gpurun_out/r02db_step python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r02db_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02db_ncu.log
tail -2 gpurun_out/r02db_fuzz_extended.txt; tail -3 gpurun_out/r02db_ncu.log
