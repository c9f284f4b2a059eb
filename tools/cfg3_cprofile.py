"""cProfile of a cold config-3 run (device noise) and of a warm second run in
the same process: where the first run's extra ~0.6 s goes (run on a GPU box)."""
import cProfile
import io
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1711_05152_b200 as P  # noqa: E402
from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402

dev = get_device()
for run in range(2):
    wl = workloads.config3(device_rng=True)
    dev.sync()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    rep = P.sparse_fft(wl.oracle, wl.cfg)
    dev.sync()
    pr.disable()
    print(f"=== run {run}: wall {time.perf_counter() - t0:.3f} s, steps {[round(x, 4) for x in rep.step_times]}")
    st = torch.cuda.memory_stats()
    print("allocator: reserved %.1f GB, peak %.1f GB, cudaMalloc retries %d, num_alloc_retries %d, segments %d" % (
        st.get("reserved_bytes.all.current", 0) / 1e9, st.get("allocated_bytes.all.peak", 0) / 1e9,
        st.get("num_alloc_retries", 0), st.get("num_alloc_retries", 0), st.get("segment.all.current", 0)))
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22)
    print(s.getvalue()[-6000:])
