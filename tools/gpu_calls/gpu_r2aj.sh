#!/bin/bash
# round 2, call AJ: N=2 bench path (2 ranks on cuda:0 over gloo: functional smoke, not a measurement),
# the reference arm, and the default bench
mkdir -p gpurun_out
export PYTHONDONTWRITEBYTECODE=1
SFFT_B200_MULTIRANK_SMOKE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/r2aj_bench_n2_smoke.json 2> gpurun_out/r2aj_bench_n2_smoke.err
echo "rc=$?" >> gpurun_out/r2aj_bench_n2_smoke.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2aj_bench_reference.json 2> gpurun_out/r2aj_bench_reference.err
timeout 900 python bench.py > gpurun_out/r2aj_bench.json 2> gpurun_out/r2aj_bench.err
