"""Host/device timeline of config-1 MR1L steps (run on a GPU box).

Wraps Device.call / download_small: for each library call records the host
time at entry and exit and a CUDA event just before the call, so the gap
between "GPU reached this point" and "host issued the call" shows where the
device idles waiting for the host."""
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
rec = []
_call, _dls = Device.call, Device.download_small


def call(self, name, *a, **k):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(self.stream)
    t0 = time.perf_counter()
    out = _call(self, name, *a, **k)
    rec.append((name, t0, time.perf_counter(), ev))
    return out


def dls(self, t):
    ev = torch.cuda.Event(enable_timing=True)
    ev.record(self.stream)
    t0 = time.perf_counter()
    out = _dls(self, t)
    rec.append(("<sync download>", t0, time.perf_counter(), ev))
    return out


PREP = "--prep" in sys.argv


def step():
    prepare = (lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z)) if PREP else None
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                       lazy_streams=True, prepare=prepare)
    run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand), prep=sch.prep)


for _ in range(5):
    step()
dev.sync()
Device.call, Device.download_small = call, dls

import paper_1711_05152_b200.mr1l as _m  # noqa: E402
import paper_1711_05152_b200._native as _n  # noqa: E402


def _wrap(mod, name):
    fn = getattr(mod, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        out = fn(*a, **k)
        rec.append((f"[host] {name}", t0, time.perf_counter(), None))
        return out
    setattr(mod, name, w)


for mod, name in ((_m, "lattice_tables"), (_m, "_sample_units"), (_m, "candidate_primes"), (_n, "query"),
                  (_m, "_attempt_streams"), (_m, "prepare_step")):
    _wrap(mod, name)
_empty = Device.empty


def empty(self, *a, **k):
    t0 = time.perf_counter()
    out = _empty(self, *a, **k)
    rec.append(("[host] empty", t0, time.perf_counter(), None))
    return out


Device.empty = empty
for it in range(3):
    rec.clear()
    dev.sync()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    h0 = time.perf_counter()
    step()
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(dev.stream)
    h1 = time.perf_counter()
    dev.sync()
    print(f"--- step {it}: device {e0.elapsed_time(e1):.3f} ms, host {1e3 * (h1 - h0):.3f} ms")
    prev_gpu = 0.0
    for name, t0, t1, ev in sorted(rec, key=lambda x: x[1]):
        if ev is None:
            print(f"  {name:28s} host@{1e3 * (t0 - h0):7.3f} dur {1e3 * (t1 - t0):6.3f}")
            continue
        g = e0.elapsed_time(ev)
        print(f"  {name:28s} host@{1e3 * (t0 - h0):7.3f} dur {1e3 * (t1 - t0):6.3f}  gpu@{g:7.3f} "
              f"(+{g - prev_gpu:6.3f})")
        prev_gpu = g
