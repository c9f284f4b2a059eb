"""8 MB pinned H2D copy time after a gap without PCIe traffic (GPU idle or
busy with a kernel during the gap): does the link slow down when idle?"""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
h = torch.empty(1000000, dtype=torch.int64, pin_memory=True).random_(0, 64)
busy = torch.empty(64 << 20, dtype=torch.float32, device=dev)


def one(gap_ms, gpu_busy):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if gpu_busy:
        while time.perf_counter() - t0 < gap_ms * 1e-3:
            busy.mul_(1.0)
            torch.cuda.synchronize()
    else:
        while time.perf_counter() - t0 < gap_ms * 1e-3:
            pass
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.to(dev, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


for _ in range(20):
    one(0, False)
for gpu_busy in (False, True):
    for gap in (0.0, 0.2, 0.5, 1.0, 2.0, 5.0, 20.0):
        ts = [one(gap, gpu_busy) for _ in range(7)]
        print(f"gap {gap:5.1f} ms {'gpu busy' if gpu_busy else 'gpu idle'}: median {np.median(ts):6.1f} us  "
              f"[{' '.join(f'{t:.0f}' for t in ts)}]")
