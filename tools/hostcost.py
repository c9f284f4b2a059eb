"""Host-side cost of individual library calls (run on a GPU box)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import _native, workloads  # noqa: E402
from paper_1711_05152_b200.device import dptr, get_device, hptr  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, lattice_tables  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand = DeviceFreqs.from_host(dev, wl.cand)
sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
ms = np.asarray(sch.primes, dtype=np.int64)
zh = np.ascontiguousarray(sch.z.astype(np.int32))
l_max = len(ms)
words = int(_native.query("sfft_alias_scratch_words", hptr(ms), l_max))
scratch = dev.empty((words,), torch.int32)
masks = dev.empty((cand.n,), torch.int64)
stats = dev.empty((2,), torch.int32)
x = dev.empty((16, 2), torch.float64)


def t(label, f, k=200):
    f()
    dev.sync()
    acc = 0.0
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        acc += time.perf_counter() - t0
        dev.sync()
    print(f"{label:40s} {1e6 * acc / k:8.2f} us")


t("ctypes abi_version", lambda: _native.query("sfft_abi_version"))
t("torch.cuda.device ctx", lambda: torch.cuda.device(0).__enter__())
t("dev.empty 100000 int64", lambda: dev.empty((100000,), torch.int64))
t("cscale n=16 (small params)", lambda: dev.call("sfft_cscale", dptr(x), 16, 1.0, 0))
t("alias_masks n=1", lambda: dev.call("sfft_alias_masks", dptr(cand.data), 1, 10, cand.kmax, hptr(ms), hptr(zh),
                                      l_max, dptr(scratch), words, dptr(masks), dptr(stats)))
t("alias_masks n=100000", lambda: dev.call("sfft_alias_masks", dptr(cand.data), cand.n, 10, cand.kmax, hptr(ms),
                                           hptr(zh), l_max, dptr(scratch), words, dptr(masks), dptr(stats)))
t("download_small", lambda: dev.download_small(stats))
L = sch.L
tabs = lattice_tables(dev, sch.m_used, sch.z_used)
t("lattice_tables (cache hit)", lambda: lattice_tables(dev, sch.m_used, sch.z_used))
t("sample_poly_scratch query", lambda: _native.query("sfft_sample_poly_scratch", hptr(tabs.ms), L, 1, 2000, 0, 0))
buf = dev.empty((L, tabs.P, 2), torch.float64)
t("bluestein", lambda: dev.call("sfft_bluestein", hptr(tabs.ms), L, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                                dptr(tabs.chirp), dptr(buf), 0, 0), k=50)
