"""Single 8 MB pinned H2D copies in the e2e pattern: which factor makes them slow
(pin_memory() vs empty(pin_memory=True), a preceding L2-flush kernel, idle gap)."""
import time

import numpy as np
import torch

dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
a_np = np.random.default_rng(0).integers(-32, 33, size=(100000, 10))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
variants = {
    "pin_memory()": torch.from_numpy(a_np).pin_memory(),
    "empty(pin)+copy": torch.empty((100000, 10), dtype=torch.int64, pin_memory=True).copy_(torch.from_numpy(a_np)),
}


def one(h, do_flush, idle_us):
    if do_flush:
        flush.zero_()
    torch.cuda.synchronize()
    if idle_us:
        t = time.perf_counter()
        while time.perf_counter() - t < idle_us * 1e-6:
            pass
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d = h.to(dev, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


for name, h in variants.items():
    assert h.is_pinned()
    for do_flush in (False, True):
        for idle in (0, 200):
            ts = [one(h, do_flush, idle) for _ in range(8)][2:]
            print(f"{name:16s} flush={do_flush!s:5s} idle={idle:3d}us: {np.median(ts):7.1f} us median "
                  f"({8 * 2**20 / np.median(ts) / 1e3:5.1f} GB/s)")
# back-to-back
h = variants["pin_memory()"]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    d = h.to(dev, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"back-to-back x10: {e0.elapsed_time(e1) * 100:.1f} us each")
