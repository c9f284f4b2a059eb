"""Wall-time spread of warm config-2 sparse_fft runs with Python's garbage
collector enabled vs disabled around each run (GPU box)."""
import gc
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import paper_1711_05152_b200 as P
    from paper_1711_05152_b200 import workloads
    from paper_1711_05152_b200.device import get_device
    dev = get_device()
    wl = workloads.config2()
    for _ in range(2):
        P.sparse_fft(wl.oracle, wl.cfg)
    dev.sync()
    out = {}
    for mode in ("gc_on", "gc_off", "gc_on", "gc_off"):
        walls = []
        for _ in range(15):
            if mode == "gc_off":
                gc.disable()
            t0 = time.perf_counter()
            P.sparse_fft(wl.oracle, wl.cfg)
            dev.sync()
            walls.append(1e3 * (time.perf_counter() - t0))
            gc.enable()
        out.setdefault(mode, []).extend(walls)
    for k, v in out.items():
        v = np.asarray(v)
        print(json.dumps({"mode": k, "median_ms": round(float(np.median(v)), 2), "max_ms": round(float(v.max()), 2),
                          "p90_ms": round(float(np.percentile(v, 90)), 2), "walls": [round(x, 2) for x in v]}))


if __name__ == "__main__":
    main()
