"""Device timeline of the head of api.reconstruct_step (terms + rows upload,
row packing) on config 1, events around each piece (run on a GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1711_05152_b200 import workloads  # noqa: E402
from paper_1711_05152_b200.device import get_device  # noqa: E402
from paper_1711_05152_b200.mr1l import DeviceFreqs  # noqa: E402

dev = get_device()
torch = dev.torch
wl = workloads.config1()
cand_host = torch.from_numpy(wl.cand).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev.device)


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(dev.stream)
    return e


for it in range(6):
    flush.zero_()
    dev.sync()
    h0 = time.perf_counter()
    e0 = ev()
    wl.oracle._dev_cache.pop(dev.index, None)
    wl.oracle.device_terms(dev)
    e1 = ev()
    h1 = time.perf_counter()
    with torch.cuda.stream(dev.stream):
        d_rows = cand_host.to(dev.device, non_blocking=True)
    e2 = ev()
    h2 = time.perf_counter()
    cand, lo, hi = DeviceFreqs.from_rows_tensor(dev, cand_host)
    e3 = ev()
    h3 = time.perf_counter()
    dev.sync()
    print(f"terms {e0.elapsed_time(e1) * 1e3:7.1f} us (host {1e6 * (h1 - h0):6.1f})  rows copy {e1.elapsed_time(e2) * 1e3:7.1f} us "
          f"(host {1e6 * (h2 - h1):6.1f})  from_rows_tensor {e2.elapsed_time(e3) * 1e3:7.1f} us (host {1e6 * (h3 - h2):6.1f})")
