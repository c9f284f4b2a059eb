"""Allocator churn of warm sparse_fft runs: segments (cudaMalloc) and frees per run (GPU box)."""
import sys, time
sys.path.insert(0, '.')
import torch
import paper_1711_05152_b200 as P
from paper_1711_05152_b200 import workloads
from paper_1711_05152_b200.device import get_device
dev = get_device()
for name, wl in (("config2", workloads.config2()), ("config4", workloads.config4())):
    P.sparse_fft(wl.oracle, wl.cfg); dev.sync()
    for k in range(3):
        s0 = torch.cuda.memory_stats()
        t0 = time.perf_counter(); P.sparse_fft(wl.oracle, wl.cfg); dev.sync(); w = time.perf_counter() - t0
        s1 = torch.cuda.memory_stats()
        d = {key: s1.get(key, 0) - s0.get(key, 0) for key in ("segment.all.allocated", "segment.all.freed", "num_alloc_retries", "allocation.all.allocated")}
        print(name, k, round(w * 1e3, 2), d, "reserved GB", round(s1["reserved_bytes.all.current"] / 2**30, 2), flush=True)
