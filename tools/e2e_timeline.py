"""Host/device timeline of api.reconstruct_step (the e2e path) on config 1."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.api import reconstruct_step  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand_host = torch.from_numpy(wl.cand).pin_memory()
rec = []


def wrap(name):
    fn = getattr(Device, name)

    def w(self, *a, **k):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        t0 = time.perf_counter()
        out = fn(self, *a, **k)
        label = a[0] if name == "call" else name
        rec.append((str(label), t0, time.perf_counter(), ev))
        return out
    setattr(Device, name, w)


for _ in range(5):
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
dev.sync()
for name in ("call", "download_small", "download_many", "upload", "empty"):
    wrap(name)
for it in range(2):
    rec.clear()
    dev.sync()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    h0 = time.perf_counter()
    reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    h1 = time.perf_counter()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(dev.stream)
    dev.sync()
    print(f"--- call {it}: host {1e3 * (h1 - h0):.3f} ms, device {e0.elapsed_time(e1):.3f} ms")
    for name, t0, t1, ev in rec:
        print(f"  {name:28s} host@{1e3 * (t0 - h0):7.3f} dur {1e3 * (t1 - t0):6.3f} gpu@{e0.elapsed_time(ev):7.3f}")
