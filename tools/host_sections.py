"""Host time per Python section of the config-1 step, warm (run on a GPU box).

Wraps the engine's functions with perf_counter timers (no profiler
overhead elsewhere) and prints, for the bench's device-resident step
(build_scheme + run_step) and for the e2e call (api.reconstruct_step), the
mean host time inside each section per call, the time spent waiting for the
GPU (synchronisations), and the remainder."""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import api, device, mr1l, workloads  # noqa: E402
from paper_1711_05152_b200 import _native  # noqa: E402

acc = defaultdict(float)
cnt = defaultdict(int)
depth = [0]


def wrap(mod, name, label=None):
    fn = getattr(mod, name)
    label = label or f"{mod.__name__.split('.')[-1]}.{name}"

    def w(*a, **k):
        t0 = time.perf_counter()
        depth[0] += 1
        try:
            return fn(*a, **k)
        finally:
            depth[0] -= 1
            acc[label] += time.perf_counter() - t0
            cnt[label] += 1
    setattr(mod, name, w)
    return fn


for name in ("build_scheme", "run_step", "prepare_step", "speculate_scheme", "_sample_units", "lattice_tables",
             "first_chunk", "apply_cap_rows"):
    if hasattr(mr1l, name):
        wrap(mr1l, name)
# api imports these names into its own namespace inside the function (from .mr1l import ...), so the
# module attributes above are what it calls
for name in ("download_small", "download_many", "download_async", "empty", "zeros", "upload", "call"):
    wrap(device.Device, name, f"Device.{name}")
_ncall = _native.call


def ncall_w(name, *a, **k):
    t0 = time.perf_counter()
    try:
        return _ncall(name, *a, **k)
    finally:
        acc["  lib:" + name] += time.perf_counter() - t0
        cnt["  lib:" + name] += 1


_native.call = ncall_w
api.build_scheme = mr1l.build_scheme  # api imported the original at module level
import torch  # noqa: E402
_sync = torch.cuda.Stream.synchronize


def sync_w(self):
    t0 = time.perf_counter()
    try:
        return _sync(self)
    finally:
        acc["(stream.synchronize)"] += time.perf_counter() - t0
        cnt["(stream.synchronize)"] += 1


torch.cuda.Stream.synchronize = sync_w
_esync = torch.cuda.Event.synchronize


def esync_w(self):
    t0 = time.perf_counter()
    try:
        return _esync(self)
    finally:
        acc["(event.synchronize)"] += time.perf_counter() - t0
        cnt["(event.synchronize)"] += 1


torch.cuda.Event.synchronize = esync_w


def report(title, reps, wall):
    print(f"=== {title}: {1e3 * wall / reps:.3f} ms host wall per call")
    for k in sorted(acc, key=lambda k: -acc[k]):
        print(f"  {k:32s} {1e6 * acc[k] / reps:9.1f} us/call  ({cnt[k] / reps:.1f} calls)")


def main():
    dev = device.get_device()
    wl = workloads.config1()
    cand = mr1l.DeviceFreqs.from_host(dev, wl.cand)
    n = len(wl.cand)

    def step():
        prep = lambda ms, z: mr1l.prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=[np.zeros(0)], d=10)  # noqa
        sch = mr1l.build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                                lazy_streams=True, prepare=prep)
        return mr1l.run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, n, defer_cap=True,
                             prep=sch.prep)
    for _ in range(5):
        step().finalize()
    dev.sync()
    acc.clear()
    cnt.clear()
    reps = 30
    t0 = time.perf_counter()
    for _ in range(reps):
        step().finalize()
        dev.sync()
    report("bench step (build_scheme + run_step, synchronised per step)", reps, time.perf_counter() - t0)

    cand_host = torch.from_numpy(wl.cand).pin_memory()
    for _ in range(5):
        api.reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    dev.sync()
    acc.clear()
    cnt.clear()
    t0 = time.perf_counter()
    for _ in range(reps):
        api.reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
    report("e2e api.reconstruct_step", reps, time.perf_counter() - t0)

    # host cost of the torch primitives the engine uses per call
    st = dev.stream
    x = dev.empty((1024,), torch.float64)
    tests = {
        "with torch.cuda.device(i)": lambda: torch.cuda.device(dev.index).__enter__() and None,
        "with torch.cuda.stream(s)": None,
        "torch.cuda.Event()": lambda: torch.cuda.Event(),
        "Event().record(s)": lambda: torch.cuda.Event().record(st),
        "torch.empty(cuda, 1 MB)": lambda: torch.empty((131072,), dtype=torch.float64, device=dev.device),
        "torch.empty(pin, 8 B)": lambda: torch.empty((8,), dtype=torch.uint8, pin_memory=True),
        "lib sfft_fft_size": lambda: _native.query("sfft_fft_size", 200000),
    }

    def stream_ctx():
        with torch.cuda.stream(st):
            pass
    tests["with torch.cuda.stream(s)"] = stream_ctx

    def dev_ctx():
        with torch.cuda.device(dev.index):
            pass
    tests["with torch.cuda.device(i)"] = dev_ctx
    print("=== torch primitives (us per op)")
    for k, f in tests.items():
        for _ in range(50):
            f()
        t0 = time.perf_counter()
        for _ in range(500):
            f()
        print(f"  {k:32s} {1e6 * (time.perf_counter() - t0) / 500:8.2f}")


if __name__ == "__main__":
    main()
