#!/bin/bash
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for ks in auto 2 3 4 5 6 7 8; do
  if [ $ks = auto ]; then timeout 300 python tools/ksplit_ab.py >> gpurun_out/r2l_ksplit.jsonl 2>&1;
  else SFFT_B200_KSPLIT=$ks timeout 300 python tools/ksplit_ab.py >> gpurun_out/r2l_ksplit.jsonl 2>&1; fi
done
