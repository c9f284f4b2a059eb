"""Per-call spread of the bench's e2e measurement (api.reconstruct_step on
pinned host rows, L2 flushed between calls, CUDA events around each call)
on a GPU box: 40 calls with the cyclic garbage collector on, then 40 with
it off."""
import gc
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.api import reconstruct_step
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    torch = dev.torch
    wl = workloads.config1()
    cand_host = torch.from_numpy(wl.cand).pin_memory()
    flush = dev.empty((64 * 1024 * 1024,), torch.float32)

    def run(k):
        out = []
        for _ in range(k):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            flush.zero_()
            dev.sync()
            a.record(dev.stream)
            reconstruct_step(cand_host, wl.oracle, b=wl.b, seed_seq=wl.lattice_seed, delta=wl.delta)
            b.record(dev.stream)
            dev.sync()
            out.append(a.elapsed_time(b))
        return np.array(out)
    run(5)
    on = run(40)
    gc.disable()
    off = run(40)
    gc.enable()
    for name, x in (("gc on", on), ("gc off", off)):
        print(json.dumps({"mode": name, "mean_ms": float(x.mean()), "median_ms": float(np.median(x)),
                          "min_ms": float(x.min()), "max_ms": float(x.max()),
                          "over_2ms": int((x > 2.0).sum()), "calls": [round(float(v), 3) for v in x]}))


if __name__ == "__main__":
    main()
