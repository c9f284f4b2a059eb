"""Host critical path of the bench's config-1 step loop: time from the alias
read-back returning on the host to the sampling launch (perf_counter stamps
around Device.download_async's waiter and Device.call); run on a GPU box."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step  # noqa: E402

dev = get_device()
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
n = len(wl.cand)
stamps = []
_call, _dla = Device.call, Device.download_async


def call(self, name, *a, **k):
    t0 = time.perf_counter()
    out = _call(self, name, *a, **k)
    stamps.append((name, t0, time.perf_counter()))
    return out


def dla(self, t, ring=8):
    w = _dla(self, t, ring)

    def wait():
        t0 = time.perf_counter()
        v = w()
        stamps.append(("wait", t0, time.perf_counter()))
        return v
    return wait


Device.call, Device.download_async = call, dla

import paper_1711_05152_b200.mr1l as _m  # noqa: E402


def _wrap(obj, name):
    fn = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        out = fn(*a, **k)
        stamps.append((f"py:{name}", t0, time.perf_counter()))
        return out
    setattr(obj, name, w)


_wrap(_m.LatticeTables, "prefix")
_wrap(_m, "_sample_units")
_wrap(_m, "run_step")
_wrap(_m, "build_scheme")
run_step = _m.run_step
build_scheme = _m.build_scheme


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
stamps.clear()
res = None
for _ in range(8):
    res = step(res)
res.finalize()
dev.sync()
t_ref = stamps[0][1]
last_wait = None
for name, t0, t1 in stamps:
    print(f"{name:28s} enter {1e6 * (t0 - t_ref):9.1f} us  dur {1e6 * (t1 - t0):7.1f} us")
    if name == "wait":
        last_wait = t1
    if name == "sfft_sample_poly_run" and last_wait is not None:
        print(f"   -> read-back to sampling launch: {1e6 * (t0 - last_wait):.1f} us host, launch call {1e6 * (t1 - t0):.1f} us")
