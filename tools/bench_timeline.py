"""GPU idle gaps of the bench's config-1 step loop (prepared steps, deferred
cap): CUDA events before/after every library call (run on a GPU box)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
n = len(wl.cand)


def step(prev=None):
    prepare = lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=[np.zeros(0)], d=10)  # noqa: E731
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                       lazy_streams=True, prepare=prepare)
    res = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, n, defer_cap=True, prep=sch.prep)
    if prev is not None:
        prev.finalize()
    return res


res = None
for _ in range(5):
    res = step(res)
res.finalize()
dev.sync()
rec = []
_call = Device.call


def call(self, name, *a, **k):
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(self.stream)
    t0 = time.perf_counter()
    out = _call(self, name, *a, **k)
    t1 = time.perf_counter()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(self.stream)
    rec.append((name, t0, t1, e0, e1))
    return out


Device.call = call
base = torch.cuda.Event(enable_timing=True)
base.record(dev.stream)
h0 = time.perf_counter()
res = None
for _ in range(4):
    res = step(res)
res.finalize()
dev.sync()
print("name                           host_start  host_dur  gpu_start  gpu_dur   gap_before")
prev_end = 0.0
for name, t0, t1, e0, e1 in rec:
    gs, ge = base.elapsed_time(e0), base.elapsed_time(e1)
    print(f"{name:30s} {1e3 * (t0 - h0):9.3f} {1e3 * (t1 - t0):9.3f} {gs:10.3f} {ge - gs:8.3f} {gs - prev_end:10.3f}")
    prev_end = ge
