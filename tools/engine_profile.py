"""Per-kernel-class device time of a full sparse_fft run (CUDA events in the library)."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1711_05152_b200 as P
from paper_1711_05152_b200 import _native, workloads
from paper_1711_05152_b200.device import get_device

dev = get_device()
for c in sys.argv[1:] or ["2", "4"]:
    wl = {"0": workloads.config0, "2": workloads.config2, "4": workloads.config4,
          "3d": lambda: workloads.config3(device_rng=True)}[c]()
    P.sparse_fft(wl.oracle, wl.cfg)
    dev.sync()
    _native.query("sfft_profile_enable", 1)
    t0 = time.perf_counter()
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    dev.sync()
    wall = time.perf_counter() - t0
    out = {}
    for cls, name in enumerate(("sample_poly", "fft", "alias", "gather")):
        tot, cnt = ctypes.c_double(), ctypes.c_int()
        _native.call("sfft_profile_collect", cls, ctypes.addressof(tot), ctypes.addressof(cnt))
        out[name] = round(tot.value, 3)
    _native.query("sfft_profile_enable", 0)
    print(wl.name, "wall_ms", round(wall * 1e3, 2), "device ms by class", out)
