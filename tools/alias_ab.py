"""K3 alias kernels A/B: mean device time of sfft_alias_masks_range over the
first chunk of lattices (library CUDA events), at config-1 size (|J| = 1e5,
d = 10) and config-3 size (|J| = 6.5e5, d = 20).  The path is chosen by
SFFT_B200_ALIAS_CLUSTER (1: cluster/DSMEM where it fits) and
SFFT_B200_ALIAS_COUNTERS (0: the 2-bit bitmaps everywhere; default: 32-bit
counters where they fit in 32 MB).  ``call_ms``: CUDA events around the whole
call (memsets included)."""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_1711_05152_b200 import _native
    from paper_1711_05152_b200.device import dptr, get_device, hptr
    from paper_1711_05152_b200.mr1l import DeviceFreqs, first_chunk
    from paper_1711_05152_b200.primes import MLConfig, primes_above
    from paper_1711_05152_b200.workloads import distinct_rows
    dev = get_device()
    torch = dev.torch
    out = {"path": "cluster" if os.environ.get("SFFT_B200_ALIAS_CLUSTER") == "1" else
           ("bitmaps" if os.environ.get("SFFT_B200_ALIAS_COUNTERS") == "0" else "counters where they fit")}
    for name, n, d in (("config1", 100_000, 10), ("config3", 650_000, 20)):
        rows = distinct_rows(np.random.default_rng(1), n, d, 32)
        cand = DeviceFreqs.from_host(dev, rows)
        cfg = MLConfig()
        L = cfg.max_lattices(n)
        ms = np.asarray(primes_above(cfg.size_lower_bound(n), L), dtype=np.int64)
        lhi = first_chunk(n, ms)
        zh = np.ascontiguousarray(np.random.default_rng(2).integers(0, ms[:, None], size=(L, d)).astype(np.int32))
        words = int(_native.query("sfft_alias_scratch_words", hptr(ms), L))
        scratch = dev.empty((words,), torch.int32)
        masks = dev.empty((n,), torch.int64)
        stats = dev.empty((2,), torch.int32)
        flush = dev.empty((64 << 20,), torch.float32)

        def run():
            dev.call("sfft_alias_masks_range", dptr(cand.data), n, d, cand.kmax, hptr(ms), hptr(zh), 0, lhi,
                     dptr(scratch), words, dptr(masks), dptr(stats))
        for _ in range(3):
            run()
        dev.sync()
        tot, cnt = ctypes.c_double(0.0), ctypes.c_int(0)
        _native.call("sfft_profile_collect", 2, ctypes.addressof(tot), ctypes.addressof(cnt))
        _native.query("sfft_profile_enable", 1)
        evs = []
        for _ in range(20):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(dev.stream)
            run()
            b.record(dev.stream)
            evs.append((a, b))
        dev.sync()
        _native.call("sfft_profile_collect", 2, ctypes.addressof(tot), ctypes.addressof(cnt))
        _native.query("sfft_profile_enable", 0)
        out[name] = {"n": n, "d": d, "lattices": lhi, "ms": tot.value / max(cnt.value, 1),
                     "call_ms": float(np.mean([a.elapsed_time(b) for a, b in evs])),
                     "masks_sum": int(dev.download(masks).view(np.uint64).sum() % (1 << 61))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
