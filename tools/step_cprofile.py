"""cProfile of the bench's config-1 step loop (L2 flush between steps, the
cap check deferred to the next step) to find where the host blocks on the
GPU (run on a GPU box)."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step, run_step  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
n = len(wl.cand)
flush = dev.empty((64 * 1024 * 1024,), torch.float32)


def step(prev=None):
    prepare = lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=[np.zeros(0)], d=10)  # noqa: E731
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64,
                       lazy_streams=True, prepare=prepare)
    res = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, n, defer_cap=True, prep=sch.prep)
    if prev is not None:
        prev.finalize()
    return sch, res


def loop(k):
    res = None
    for _ in range(k):
        flush.zero_()
        sch, res = step(res)
    res.finalize()
    dev.sync()


loop(5)
pr = cProfile.Profile()
pr.enable()
loop(20)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumtime").print_stats(40)

# which torch.empty blocks: time every call, print the slow ones' call sites
import time  # noqa: E402
import traceback  # noqa: E402
_empty = torch.empty
slow = []


def empty_w(*a, **k):
    t0 = time.perf_counter()
    out = _empty(*a, **k)
    dt = time.perf_counter() - t0
    if dt > 1e-4:
        slow.append((dt, a, {kk: str(v) for kk, v in k.items()}, traceback.format_stack(limit=4)[:-1]))
    return out


tot = [0.0]


def empty_t(*a, **k):
    t0 = time.perf_counter()
    out = empty_w(*a, **k)
    tot[0] += time.perf_counter() - t0
    return out


torch.empty = empty_t
for rep in range(3):
    tot[0] = 0.0
    t0 = time.perf_counter()
    m0 = torch.cuda.memory_stats()
    loop(20)
    m1 = torch.cuda.memory_stats()
    print({k: m1.get(k, 0) - m0.get(k, 0) for k in ("num_device_alloc", "num_device_free", "num_alloc_retries",
                                                  "num_sync_all_streams", "allocation.all.allocated")},
          "reserved GB", m1.get("reserved_bytes.all.current", 0) / 1e9,
          "allocated GB", m1.get("allocated_bytes.all.current", 0) / 1e9,
          "inactive split GB", m1.get("inactive_split_bytes.all.current", 0) / 1e9)
    print(f"loop(20): {1e3 * (time.perf_counter() - t0):.2f} ms, torch.empty total {1e3 * tot[0]:.2f} ms")
for dt, a, k, stack in slow[:6]:
    print(f"{dt * 1e3:.3f} ms", a, k)
    print("".join(stack))
print("slow calls:", len(slow))
