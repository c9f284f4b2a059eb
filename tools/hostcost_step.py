"""Host cost of every library call of the bench's config-1 step: the calls of
one step are captured and each is replayed k times (host time per call, GPU
synchronised between replays); plus the Python time of build_scheme/run_step
outside the library calls.  Run on a GPU box."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import _native, workloads  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step  # noqa: E402

dev = get_device()
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
n = len(wl.cand)
calls = []
_call = Device.call
capture = [False]
lib_time = [0.0]


def call(self, name, *a, **k):
    t0 = time.perf_counter()
    out = _call(self, name, *a, **k)
    lib_time[0] += time.perf_counter() - t0
    if capture[0]:
        calls.append((name, a, k))
    return out


Device.call = call


def step():
    prepare = lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=[np.zeros(0)], d=10)  # noqa: E731
    t0 = time.perf_counter()
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                       lazy_streams=True, prepare=prepare)
    t1 = time.perf_counter()
    res = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, n, defer_cap=True, prep=sch.prep)
    t2 = time.perf_counter()
    res.finalize()
    dev.sync()
    return t1 - t0, t2 - t1, res


for _ in range(5):
    step()
acc = np.zeros(2)
lib = 0.0
K = 20
for _ in range(K):
    lib_time[0] = 0.0
    a, b, _ = step()
    acc += (a, b)
    lib += lib_time[0]
print(f"build_scheme {1e6 * acc[0] / K:.1f} us host, run_step {1e6 * acc[1] / K:.1f} us host, "
      f"library calls inside {1e6 * lib / K:.1f} us")
capture[0] = True
keep = step()
capture[0] = False
for name, a, k in calls:
    if name == "sfft_alias_masks":
        continue
    dev.sync()
    tot = 0.0
    for _ in range(20):
        t0 = time.perf_counter()
        _call(dev, name, *a, **k)
        tot += time.perf_counter() - t0
        dev.sync()
    print(f"{name:28s} {1e6 * tot / 20:8.2f} us host per call")
t0 = time.perf_counter()
for _ in range(1000):
    _native.query("sfft_abi_version")
print(f"ctypes no-arg call {1e3 * (time.perf_counter() - t0):.2f} us")
