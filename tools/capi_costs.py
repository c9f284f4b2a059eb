"""Host cost of the C-ABI entry points of a config-1 step (GPU box): each call
timed in a tight loop (ctypes + C++ + CUDA launch API), 200 calls, the stream
drained every 20 so the launch queue stays short."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_1711_05152_b200 import _native, workloads
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    from paper_1711_05152_b200.mr1l import DeviceFreqs, build_scheme, prepare_step
    dev = get_device()
    wl = workloads.config1()
    cand = DeviceFreqs.from_host(dev, wl.cand)
    tails = [np.zeros(0)]
    sch = build_scheme(dev, cand, wl.b, np.random.SeedSequence(wl.lattice_seed), box_extent=64, lazy_streams=True,
                       prepare=lambda ms, z: prepare_step(dev, wl.oracle, cand, 1, ms, z, tails=tails, d=10))
    prep = sch.prep
    tabs = prep.tabs
    ms = np.ascontiguousarray(tabs.ms)
    zs = np.ascontiguousarray(tabs.zs)
    L = len(ms)
    hf, cf = wl.oracle.device_terms(dev)
    cprime, rres, rj, scratch = prep.poly
    anchor = np.zeros(1)
    words = int(_native.query("sfft_alias_scratch_words", hptr(ms), L))
    ascr = dev.empty((words,), dev.torch.int32)
    masks = dev.empty((cand.n,), dev.torch.int64)
    stats = dev.empty((2,), dev.torch.int32)
    st = dev.sh
    out = {}

    def t(name, fn, reps=200):
        for _ in range(5):
            fn()
        dev.sync()
        tot = 0.0
        for k in range(reps):
            a = time.perf_counter()
            fn()
            tot += time.perf_counter() - a
            if k % 20 == 19:
                dev.sync()
        dev.sync()
        out[name] = round(1e6 * tot / reps, 2)

    t("query sfft_fft_size (ctypes floor)", lambda: _native.query("sfft_fft_size", 200000))
    t("sfft_sample_poly_scratch (plan only)",
      lambda: _native.query("sfft_sample_poly_scratch", hptr(ms), L, 1, wl.oracle.s, 0, 0))
    t("sfft_alias_masks_range (2 memsets + 2 kernels)",
      lambda: _native.call("sfft_alias_masks_range", dptr(cand.data), cand.n, 10, 64, hptr(ms), hptr(zs), 0, L,
                           dptr(ascr), words, dptr(masks), dptr(stats), st))
    t("sfft_sample_poly_prepare (plan + 3 kernels)",
      lambda: _native.call("sfft_sample_poly_prepare", dptr(hf), dptr(cf), wl.oracle.s, 10, 10, hptr(ms), hptr(zs), L,
                           hptr(anchor), 1, dptr(cprime), dptr(rres), dptr(rj), dptr(tabs.tw), dptr(scratch),
                           int(scratch.shape[0]), 0, st), reps=50)
    buf = dev.empty((L, tabs.P, 2), dev.torch.float64)
    t("sfft_bluestein (3 kernels)",
      lambda: _native.call("sfft_bluestein", hptr(ms), L, 1, tabs.P, dptr(tabs.ftab), dptr(tabs.bhat),
                           dptr(tabs.chirp), dptr(buf), 0, 0, st), reps=50)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
