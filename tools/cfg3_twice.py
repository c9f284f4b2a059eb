"""Config 3 (device noise) run twice in one process: per-step wall times of
the first (allocator / table cold) and the second run (run on a GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
for run in range(2):
    wl = workloads.config3(device_rng=True)
    dev.sync()
    t0 = time.perf_counter()
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    dev.sync()
    wall = time.perf_counter() - t0
    st = getattr(rep, "step_times", None)
    print(f"run {run}: wall {wall:.3f} s, steps {[round(x, 4) for x in st] if st is not None else '-'}", flush=True)
