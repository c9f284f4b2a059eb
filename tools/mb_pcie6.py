"""The e2e head pattern (L2 flush, oracle terms re-upload, 8 MB rows copy) with
one factor removed at a time, to find what makes the rows copy slow."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
rows_a = torch.from_numpy(wl.cand).pin_memory()
rows_b = torch.empty(wl.cand.shape, dtype=torch.int64, pin_memory=True)
rows_b.copy_(torch.from_numpy(wl.cand))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev.device)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(dev.stream)
    return e


def run(rows, do_flush, do_terms, reps=8):
    ts = []
    for _ in range(reps):
        if do_flush:
            with torch.cuda.stream(dev.stream):
                flush.zero_()
        dev.sync()
        if do_terms:
            wl.oracle._dev_cache.pop(dev.index, None)
            wl.oracle.device_terms(dev)
        e1 = ev()
        with torch.cuda.stream(dev.stream):
            rows.to(dev.device, non_blocking=True)
        e2 = ev()
        dev.sync()
        ts.append(e1.elapsed_time(e2) * 1e3)
    return np.median(ts[2:]), ts


for name, rows in (("pin_memory()", rows_a), ("empty(pin)+copy_", rows_b)):
    for do_flush in (True, False):
        for do_terms in (True, False):
            med, ts = run(rows, do_flush, do_terms)
            print(f"{name:18s} flush={do_flush!s:5s} terms={do_terms!s:5s}: {med:6.1f} us  "
                  f"[{' '.join(f'{t:.0f}' for t in ts)}]")
