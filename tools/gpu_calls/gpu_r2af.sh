#!/bin/bash
# round 2, call AF: engine overlap A/B (configs 0, 2, 2s, 4), twice each
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
for rep in 1 2; do
for ov in 1 0; do
SFFT_B200_ENGINE_OVERLAP=$ov timeout 600 python tools/run_configs.py 0 2 2s 4 > gpurun_out/r2af_configs_ov${ov}_$rep.jsonl 2>&1
done
done
