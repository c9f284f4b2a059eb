#!/bin/bash
# round 2, call DC: ncu --set full of the config-1 step kernels of the final code; raw and details pages exported on the
# box (the report with sources exceeds the 64 MiB copy-back limit and stays there)
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r02dc_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"sample_poly_tcp|fft_colx|fft_row2048|gather_kernel|alias_c|poly_bpanel" --launch-skip 8 --launch-count 10 \
  -o /tmp/r02dc_step python tools/profile_step.py --warmup 1 --steps 1 > gpurun_out/r02dc_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02dc_ncu.log
ncu -i /tmp/r02dc_step.ncu-rep --page raw --csv > gpurun_out/r02dc_step_raw.csv 2>/dev/null
ncu -i /tmp/r02dc_step.ncu-rep --page details --csv > gpurun_out/r02dc_step_details.csv 2>/dev/null
ls -la /tmp/r02dc_step.ncu-rep gpurun_out/r02dc_*; rm -f /tmp/r02dc_step.ncu-rep
