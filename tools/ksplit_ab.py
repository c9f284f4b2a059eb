"""K1 K-split A/B on config 1: mean device time of the sampling class
(library CUDA events) per SFFT_B200_KSPLIT setting (run once per setting)."""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_1711_05152_b200 import _native, workloads
    from paper_1711_05152_b200.device import get_device
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, run_step
    dev = get_device()
    wl = workloads.config1()
    cand = DeviceFreqs.from_host(dev, wl.cand)
    flush = dev.empty((64 << 20,), dev.torch.float32)
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64)
    for _ in range(3):
        run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand))
    dev.sync()
    tot, cnt = ctypes.c_double(0.0), ctypes.c_int(0)
    _native.call("sfft_profile_collect", 0, ctypes.addressof(tot), ctypes.addressof(cnt))
    _native.query("sfft_profile_enable", 1)
    for _ in range(10):
        flush.zero_()
        res = run_step(dev, wl.oracle, cand, sch, [np.zeros(0)], 10, wl.delta, len(wl.cand))
    dev.sync()
    _native.call("sfft_profile_collect", 0, ctypes.addressof(tot), ctypes.addressof(cnt))
    _native.query("sfft_profile_enable", 0)
    coef = dev.download(res.coef[0])
    err = np.linalg.norm(coef[:, 0] + 1j * coef[:, 1] - wl.truth_coef) / np.linalg.norm(wl.truth_coef)
    print(json.dumps({"ksplit": os.environ.get("SFFT_B200_KSPLIT", "auto"), "k1_ms": tot.value / max(cnt.value, 1),
                      "err": err}))


if __name__ == "__main__":
    main()
