"""Where the host spends a sparse_fft run (config 2): wall time of every
library call and sync, grouped by call name (run on a GPU box)."""
import collections
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import Device, get_device  # noqa: E402

dev = get_device()
wl = workloads.config2() if len(sys.argv) < 2 or sys.argv[1] == "2" else workloads.config4()
P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
acc = collections.defaultdict(lambda: [0, 0.0])
for name in ("call", "download_small", "download_many", "download", "upload", "empty", "zeros"):
    fn = getattr(Device, name)

    def w(self, *a, _fn=fn, _name=name, **k):
        t0 = time.perf_counter()
        out = _fn(self, *a, **k)
        key = f"call:{a[0]}" if _name == "call" else _name
        acc[key][0] += 1
        acc[key][1] += time.perf_counter() - t0
        return out
    setattr(Device, name, w)
dev.sync()
t0 = time.perf_counter()
rep = P.sparse_fft(wl.oracle, wl.cfg)
dev.sync()
wall = time.perf_counter() - t0
tot = sum(v[1] for v in acc.values())
print(f"wall {wall * 1e3:.2f} ms; inside library calls/syncs {tot * 1e3:.2f} ms; "
      f"other host {1e3 * (wall - tot):.2f} ms")
for k, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {k:34s} n={n:5d}  {t * 1e3:8.3f} ms")
